export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "half or 5" -p no:cacheprovider 2>&1 | tail -1
timeout 900 python tools/cosched.py --levels auto --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_h2b.log 2>&1
grep levels gpurun_out/r02_cosched_h2b.log | cut -c1-450
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"half2" -c 1 python tools/ncu_step.py --config c3 --matvecs 1 2>&1 | grep -E "half2|duration|fp64" | head -5
