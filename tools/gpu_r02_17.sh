export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "half or 5" -p no:cacheprovider > gpurun_out/r02_half_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_half_tests.log
tail -3 gpurun_out/r02_half_tests.log
timeout 900 python tools/cosched.py --levels 011102,011152,011552,015152,011112 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_half.log 2>&1
grep levels gpurun_out/r02_cosched_half.log | cut -c1-420
