export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"half2" -c 1 -o /tmp/h2 -f python tools/ncu_step.py --config c3 --matvecs 1 > gpurun_out/r02_c3_h2_ncu.log 2>&1
ncu -i /tmp/h2.ncu-rep --page details --csv > gpurun_out/r02_c3_h2_details.csv 2>/dev/null
ncu -i /tmp/h2.ncu-rep --page raw --csv > gpurun_out/r02_c3_h2_raw.csv 2>/dev/null
ncu -i /tmp/h2.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/r02_c3_h2_sass.csv.gz
