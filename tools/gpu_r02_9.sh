export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "pair or 3" -p no:cacheprovider > gpurun_out/r02_pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pair_tests.log
tail -3 gpurun_out/r02_pair_tests.log
for v in A B C D; do
  H3D_LIB_PATH=tools/lib_p$v/libh3d_b200.so timeout 300 python tools/cosched.py --levels 011132 --tunes "skip=400;skip=0" --steps 40 > gpurun_out/r02_pair_$v.log 2>&1
  echo "== $v"; grep levels gpurun_out/r02_pair_$v.log | cut -c1-110; grep levels gpurun_out/r02_pair_$v.log | grep -o "pair=[0-9.@]*"
done
