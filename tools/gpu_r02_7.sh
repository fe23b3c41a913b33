export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -c 1 -o /tmp/fv2 -f python tools/ncu_step.py --config c3 --matvecs 1 --levels 011142 > gpurun_out/r02_c3_fused_v2.log 2>&1
ncu -i /tmp/fv2.ncu-rep --page details --csv > gpurun_out/r02_c3_fused_v2_details.csv 2>/dev/null
ncu -i /tmp/fv2.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/r02_c3_fused_v2_sass.csv.gz
ls -la gpurun_out
