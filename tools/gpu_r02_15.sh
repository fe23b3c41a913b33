export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu3.log
tail -3 gpurun_out/r02_pytest_gpu3.log
timeout 900 python tools/cosched.py --levels auto,011112 --tunes "sol=2;sol=4" --steps 50 > gpurun_out/r02_cosched_sol2.log 2>&1
grep levels gpurun_out/r02_cosched_sol2.log | sed 's/power_max.*solve=/ solve=/' | cut -c1-140
