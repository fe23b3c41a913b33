export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -o gpurun_out/r02_c3_fused_v1 -f python tools/ncu_step.py --config c3 --matvecs 1 --levels 011142 > gpurun_out/r02_c3_fused_v1.log 2>&1
tail -3 gpurun_out/r02_c3_fused_v1.log
