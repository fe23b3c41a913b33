export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python tools/cosched.py --config c4 --levels auto,015152,010152,015102 --tunes "graphs=1" --steps 50 > gpurun_out/r02_half_c4.log 2>&1
timeout 600 python tools/cosched.py --config c2 --levels auto,01152,01102 --tunes "graphs=1" --steps 100 > gpurun_out/r02_half_c2.log 2>&1
timeout 900 python tools/cosched.py --config c5 --levels auto,0151152,0101152,0151102 --tunes "graphs=1" --steps 20 > gpurun_out/r02_half_c5.log 2>&1
grep levels gpurun_out/r02_half_c4.log gpurun_out/r02_half_c2.log gpurun_out/r02_half_c5.log | cut -c1-150
