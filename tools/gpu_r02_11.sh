export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python tools/build_probe.py --config c3 --builds 3 --tunes ";acat2=256" > gpurun_out/r02_build_acab.log 2>&1
cat gpurun_out/r02_build_acab.log
