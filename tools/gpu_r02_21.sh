H3D_TUNE=half_search=1 timeout 600 python tools/model_print.py c5 > gpurun_out/r02_model_c5.log 2>&1; tail -2 gpurun_out/r02_model_c5.log
H3D_TUNE=half_search=1 timeout 600 python tools/model_print.py c3 > gpurun_out/r02_model_c3h.log 2>&1; tail -1 gpurun_out/r02_model_c3h.log
timeout 900 python tools/cosched.py --config c5 --levels 0155112,0151152,0101112,0151112 --tunes "graphs=1" --steps 15 > gpurun_out/r02_half_c5b.log 2>&1
grep levels gpurun_out/r02_half_c5b.log | cut -c1-150
