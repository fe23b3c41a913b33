export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu2.log
tail -4 gpurun_out/r02_pytest_gpu2.log
timeout 600 python tools/build_probe.py --config c3 --builds 3 > gpurun_out/r02_build_c3b.log 2>&1
timeout 600 python tools/build_probe.py --config c4 --builds 2 >> gpurun_out/r02_build_c3b.log 2>&1
cat gpurun_out/r02_build_c3b.log
