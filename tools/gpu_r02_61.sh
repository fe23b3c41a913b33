export PATH=/usr/local/cuda/bin:$PATH
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/r02_f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_f_pytest_gpu.log; grep -a passed gpurun_out/r02_f_pytest_gpu.log | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/r02_f_bench_c3.json 2> gpurun_out/r02_f_bench_c3.err; echo "c3 rc=$?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/r02_f_bench_c3.json"))
print(round(d["value"],2), round(d["ms_per_step"],3), round(d["e2e"]["value"],2), d["roofline"]["kernel"], d["roofline"]["frac"], d["detail"]["step_roofline"]["frac"], d["cpu_baseline"]["value"], d["clocks"])
print({k:(v["ms"],v.get("frac_of_operand_bound")) for k,v in d["detail"]["kernels"].items()})
PY
