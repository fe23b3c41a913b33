export PATH=/usr/local/cuda/bin:$PATH
for c in c3 c4 c5; do
echo "== $c product (4 CTAs, 122 regs)"; timeout 600 python tools/cosched.py --config $c --steps 50 --tunes "skip=0;p2p=5" 2>&1 | grep levels | cut -c1-400
echo "== $c half2 at 96 regs"; H3D_LIB_PATH=tools/lib_pB/libh3d_b200.so timeout 600 python tools/cosched.py --config $c --steps 50 --tunes "skip=0;p2p=5" 2>&1 | grep levels | cut -c1-400
done > gpurun_out/r02_cosched_half5.log 2>&1
cat gpurun_out/r02_cosched_half5.log
