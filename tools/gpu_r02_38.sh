export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python bench.py > gpurun_out/r02_final_bench_c3.json 2> gpurun_out/r02_final_bench_c3.err; echo "c3 rc=$?"
for c in c2 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_final_bench_$c.json 2> gpurun_out/r02_final_bench_$c.err; echo "$c rc=$?"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_final_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_final_c3_launches_bench.log 2>&1; echo "launches rc=$?"
