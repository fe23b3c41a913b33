export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "fused or 4" -p no:cacheprovider > gpurun_out/r02_fused_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_fused_tests.log
tail -3 gpurun_out/r02_fused_tests.log
timeout 600 python tools/cosched.py --levels 011142 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_fused.log 2>&1
grep levels gpurun_out/r02_cosched_fused.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -o gpurun_out/r02_c3_fused_v2 -f python tools/ncu_step.py --config c3 --matvecs 1 --levels 011142 > gpurun_out/r02_c3_fused_v2.log 2>&1
