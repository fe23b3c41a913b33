export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "stored_direct or cached_and or bitwise" -p no:cacheprovider > gpurun_out/r02_nfd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_nfd_tests.log
tail -3 gpurun_out/r02_nfd_tests.log
timeout 900 python tools/cosched.py --levels auto --tunes "nfd=0;nfd=1;nfd=1,nfc=2;nfd=1,nf=0" --steps 50 > gpurun_out/r02_cosched_nfd.log 2>&1
grep levels gpurun_out/r02_cosched_nfd.log | cut -c1-420
