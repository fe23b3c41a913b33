export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"p2_near" -c 1 -o gpurun_out/r02_near_c5 -f python tools/ncu_step.py --config c5 --matvecs 1 > gpurun_out/r02_near_c5_ncu.log 2>&1; echo "ncu rc=$?"
