export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "pair or 3" -p no:cacheprovider > gpurun_out/r02_pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pair_tests.log
tail -3 gpurun_out/r02_pair_tests.log
timeout 600 python tools/cosched.py --levels 011102,011132 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_pair2.log 2>&1
grep levels gpurun_out/r02_cosched_pair2.log
timeout 900 ncu --set full --clock-control none -k regex:pair_kernel -c 1 -o /tmp/p2 -f python tools/ncu_step.py --config c3 --matvecs 1 --levels 011132 > gpurun_out/r02_c3_pair2.log 2>&1
ncu -i /tmp/p2.ncu-rep --page details --csv > gpurun_out/r02_c3_pair2_details.csv 2>/dev/null
