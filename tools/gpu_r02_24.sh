export PATH=/usr/local/cuda/bin:$PATH
H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so timeout 600 python tools/cosched.py --levels auto --tunes "skip=0;skip=10;skip=400;skip=256;skip=266;nf=0;p2p=3;p2p=5;p1p=5;nfc=2" --steps 50 > gpurun_out/r02_cosched_half_lanes.log 2>&1
grep levels gpurun_out/r02_cosched_half_lanes.log | cut -c1-420
