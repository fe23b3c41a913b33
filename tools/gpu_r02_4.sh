export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "fused or 4" -p no:cacheprovider > gpurun_out/r02_fused_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_fused_tests.log
tail -5 gpurun_out/r02_fused_tests.log
timeout 600 python tools/cosched.py --levels 011102,011142,011112 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_fused.log 2>&1
grep levels gpurun_out/r02_cosched_fused.log
