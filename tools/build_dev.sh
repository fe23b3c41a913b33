#!/bin/bash
# Developer build of the product library with -DH3D_DEVTOOLS (H3D_TUNE skip
# masks) into tools/lib_dev/ (git-ignored). Never the product path.
set -e
cd "$(dirname "$0")/../paper_2307_16303_b200/csrc"
OUT=../../tools/${DEV_OUT:-lib_dev}
mkdir -p $OUT/obj
NV="/usr/local/cuda/bin/nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr -DH3D_DEVTOOLS $EXTRA"
pids=()
for f in tree lists aca matvec pair fused gmres engine; do $NV -c $f.cu -o $OUT/obj/$f.o & pids+=($!); done
for f in capi planner nccl_dyn ie; do $NV -x cu -c $f.cpp -o $OUT/obj/$f.o & pids+=($!); done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libh3d_b200.so $OUT/obj/*.o -ldl
echo built $OUT/libh3d_b200.so
