export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q -k "split or 6" -p no:cacheprovider 2>&1 | grep -E "FAILED|Error|assert |^E " | head -20
