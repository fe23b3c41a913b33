export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "clustered or cached_and or stored_direct" 2>&1 | tail -8
