export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --config c3 --steps 50 --tunes "skip=0;nf=2;nf=1" > gpurun_out/r02_cosched_p1s4.log 2>&1; echo rc=$?
cut -c1-420 gpurun_out/r02_cosched_p1s4.log
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/r02_c_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_c_pytest_gpu.log
