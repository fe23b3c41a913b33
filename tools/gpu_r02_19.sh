for c in c2 c3 c4; do echo "== $c"; timeout 300 python tools/model_print.py $c > gpurun_out/r02_model_$c.log 2>&1; grep chosen gpurun_out/r02_model_$c.log; done
