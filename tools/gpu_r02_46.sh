export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"p2_near|half2" -c 2 -o gpurun_out/r02_near_half -f python tools/ncu_step.py --config c3 --matvecs 1 > gpurun_out/r02_near_half_ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/r02_near_half.ncu-rep
