export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --levels 011102,010112,001102,010102 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_modes2.log 2>&1
grep levels gpurun_out/r02_cosched_modes2.log | cut -c1-400
