export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --levels auto,011552,015552,011502,015152 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_half3.log 2>&1
grep levels gpurun_out/r02_cosched_half3.log | cut -c1-480
