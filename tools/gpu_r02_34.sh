export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 python tools/cosched.py --levels auto --tunes "graphs=1;nf=0" --steps 50 > gpurun_out/r02_cosched_db.log 2>&1
grep levels gpurun_out/r02_cosched_db.log | cut -c1-450
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"p1_proxy|p2_proxy|half2" -c 3 python tools/ncu_step.py --config c3 --matvecs 1 2>&1 | grep -E "proxy|half2|duration|fp64" | head -12
