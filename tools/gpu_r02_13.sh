export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv
timeout 900 python tools/build_probe.py --config c3 --builds 6 > gpurun_out/r02_build_var.log 2>&1
cat gpurun_out/r02_build_var.log
