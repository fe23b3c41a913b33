export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --levels auto,011112 --tunes "sol=1;sol=2;sol=3;sol=4;sol=6" --steps 50 > gpurun_out/r02_cosched_sol.log 2>&1
grep levels gpurun_out/r02_cosched_sol.log | sed 's/power_max.*solve=/ solve=/' | cut -c1-140
