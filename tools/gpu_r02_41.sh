export PATH=/usr/local/cuda/bin:$PATH
H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so timeout 900 python tools/cosched.py --config c3 --steps 50 --tunes "skip=0;h2w=0;skip=2;skip=2,h2w=0" > gpurun_out/r02_cosched_h2w.log 2>&1; echo rc=$?
cat gpurun_out/r02_cosched_h2w.log
