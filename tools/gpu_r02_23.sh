export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu5.log
tail -3 gpurun_out/r02_pytest_gpu5.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python tools/build_probe.py --config c3 --builds 4 2>&1 | tail -3
