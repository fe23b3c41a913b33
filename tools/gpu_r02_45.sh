export PATH=/usr/local/cuda/bin:$PATH
H3D_LIB_PATH=tools/lib_pA/libh3d_b200.so timeout 900 python tools/cosched.py --config c3 --steps 50 --tunes "p1s=2,p2s=2;p1s=2,p2s=2,p1p=3,p2p=3;p1s=1,p2s=1;p1s=2,p2s=1;p1s=1,p2s=2" > gpurun_out/r02_cosched_kstages2.log 2>&1; echo rc=$?
cut -c1-420 gpurun_out/r02_cosched_kstages2.log
