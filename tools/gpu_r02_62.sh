export PATH=/usr/local/cuda/bin:$PATH
for c in c4 c5 c2 c3; do
timeout 900 python tools/cosched.py --config $c --steps 50 --tunes "skip=0;skip=0" 2>&1 | grep levels | cut -c1-400
done > gpurun_out/r02_cosched_nearrows.log 2>&1
cat gpurun_out/r02_cosched_nearrows.log
timeout 900 python -m pytest tests -m gpu -x -q -k "golden or clustered or cached or stored or determin or shard or kernels" 2>&1 | tail -3
