export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_end2_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_end2_smoke.log
timeout 1200 python bench.py > gpurun_out/r02_end2_bench_c3.json 2> gpurun_out/r02_end2_bench_c3.err; echo "c3 rc=$?"
for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_end2_bench_$c.json 2> gpurun_out/r02_end2_bench_$c.err; echo "$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_end2_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_end2_c3_launches_bench.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none -k regex:"p1_stream|p2_stream|p1_proxy|p2_proxy|half2|p2_near|proxy_solve|combine" -c 8 -o /tmp/fin -f python tools/ncu_step.py --config c3 --matvecs 1 > gpurun_out/r02_end2_c3_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/fin.ncu-rep --page raw --csv > gpurun_out/r02_end2_c3_full_raw.csv 2>/dev/null
python - <<'PY'
import json
for c in ("c2","c3","c4","c5"):
    try:
        d=json.load(open(f"gpurun_out/r02_end2_bench_{c}.json"))
        print(c, round(d["value"],2), round(d["ms_per_step"],3), round(d["e2e"]["value"],2), d["roofline"]["kernel"], d["roofline"]["frac"], d["detail"]["step_roofline"]["frac"], d["clocks"])
    except Exception as e:
        print(c, "failed", e)
PY
