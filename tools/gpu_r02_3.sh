export PATH=/usr/local/cuda/bin:$PATH
export H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so
timeout 900 python tools/cosched.py --levels 011102,011132,011332,011112,013332 --tunes "skip=0;skip=400;skip=10" > gpurun_out/r02_cosched_pair.log 2>&1
timeout 300 python tools/cosched.py --levels 011132 --tunes "skip=0,pps=1;skip=0,pps=3;skip=0,p1p=3,p2p=3" >> gpurun_out/r02_cosched_pair.log 2>&1
grep levels gpurun_out/r02_cosched_pair.log | cut -c1-150
