export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --levels auto --tunes "graphs=1;nf=0;p2p=5;p2p=3;nfc=2;nf=0,p2c=2;nf=0,p2c=3" --steps 50 > gpurun_out/r02_cosched_h2c.log 2>&1
grep levels gpurun_out/r02_cosched_h2c.log | cut -c1-450
