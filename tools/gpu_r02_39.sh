export PATH=/usr/local/cuda/bin:$PATH
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/r02_re_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_re_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02_re_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/r02_re_bench_c3.json 2> gpurun_out/r02_re_bench_c3.err; echo "c3 rc=$?"; cat gpurun_out/r02_re_bench_c3.json
