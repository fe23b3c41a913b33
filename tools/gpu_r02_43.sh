export PATH=/usr/local/cuda/bin:$PATH
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/r02_b_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_b_pytest_gpu.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/r02_b_bench_c3.json 2> gpurun_out/r02_b_bench_c3.err; echo "c3 rc=$?"
for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_b_bench_$c.json 2> gpurun_out/r02_b_bench_$c.err; echo "$c rc=$?"; done
python - <<'PY'
import json
for c in ("c2","c3","c4","c5"):
    try:
        d=json.load(open(f"gpurun_out/r02_b_bench_{c}.json"))
        print(c, round(d["value"],2), d["ms_per_step"], d["e2e"]["value"], {k:(v["ms"],v["start_ms"]) for k,v in d["detail"]["kernels"].items()})
    except Exception as e:
        print(c, "failed", e)
PY
