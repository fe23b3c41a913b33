export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python tools/cosched.py --config c3 --steps 50 --levels "auto,011552,015152,015552,011052" > gpurun_out/r02_cosched_levels.log 2>&1; echo rc=$?
cut -c1-400 gpurun_out/r02_cosched_levels.log
