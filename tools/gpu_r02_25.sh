export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"p2_proxy|p2_near|p1_proxy" -c 3 -o /tmp/fp -f python tools/ncu_step.py --config c3 --matvecs 1 > gpurun_out/r02_c3_fp64_ncu.log 2>&1
ncu -i /tmp/fp.ncu-rep --page details --csv > gpurun_out/r02_c3_fp64_details.csv 2>/dev/null
ncu -i /tmp/fp.ncu-rep --page raw --csv > gpurun_out/r02_c3_fp64_raw.csv 2>/dev/null
ncu -i /tmp/fp.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/r02_c3_fp64_sass.csv.gz
ls -la gpurun_out | tail -4
