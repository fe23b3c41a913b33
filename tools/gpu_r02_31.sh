export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "split or 6" -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/cosched.py --levels 011152,066652,016652,011652,066152 --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_split.log 2>&1
grep levels gpurun_out/r02_cosched_split.log | cut -c1-480
