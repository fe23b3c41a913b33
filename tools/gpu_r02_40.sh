export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python tools/cosched.py --config c3 --steps 50 --tunes "skip=0;p1p=5,p2p=5;nfc=2;p1p=5,p2p=5,nfc=2" > gpurun_out/r02_cosched_timeline.log 2>&1; echo rc=$?
cat gpurun_out/r02_cosched_timeline.log
