set -x
export PATH=/usr/local/cuda/bin:$PATH
H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so timeout 600 python tools/cosched.py --tunes "skip=0;skip=400;skip=10;skip=2;skip=8;skip=144;skip=256;skip=402" > gpurun_out/r02_cosched.log 2>&1
H3D_LIB_PATH=tools/lib_dev/libh3d_b200.so timeout 300 python tools/cosched.py --tunes "skip=0;skip=400;skip=10" --gap-ms 5 --steps 40 >> gpurun_out/r02_cosched.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_c3_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c3_launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:aca_kernel -c 6 -o gpurun_out/r02_c3_aca -f python tools/ncu_step.py --config c3 --matvecs 0 > gpurun_out/r02_c3_aca.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:proxy_solve -c 1 -o gpurun_out/r02_c3_solve -f python tools/ncu_step.py --config c3 --matvecs 1 > gpurun_out/r02_c3_solve.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:proxy_solve -c 1 -o gpurun_out/r02_c4_solve -f python tools/ncu_step.py --config c4 --matvecs 1 > gpurun_out/r02_c4_solve.log 2>&1
ls -la gpurun_out
