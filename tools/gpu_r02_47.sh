export PATH=/usr/local/cuda/bin:$PATH
for c in c3 c4 c5 c2; do
for lib in lib_pA lib_pB lib_pA lib_pB; do
echo "== $c $lib"
H3D_LIB_PATH=tools/$lib/libh3d_b200.so timeout 600 python tools/cosched.py --config $c --steps 50 --tunes "skip=0" 2>&1 | grep levels | cut -c1-420
done; done > gpurun_out/r02_cosched_p2p_regs.log 2>&1
cat gpurun_out/r02_cosched_p2p_regs.log
