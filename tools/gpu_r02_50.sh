export PATH=/usr/local/cuda/bin:$PATH
for c in c4 c2 c5 c3; do
echo "== $c"
timeout 900 python tools/cosched.py --config $c --steps 50 --tunes "nfc=1;nfc=2;nfc=1;nfc=2" 2>&1 | grep levels | cut -c1-400
done > gpurun_out/r02_cosched_nfc.log 2>&1
cat gpurun_out/r02_cosched_nfc.log
timeout 600 python -m pytest tests -m gpu -x -q -k "golden or determin or shard" 2>&1 | tail -3
