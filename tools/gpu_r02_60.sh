export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -x -q -k "clustered" 2>&1 | tail -25
