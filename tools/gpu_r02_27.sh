export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu6.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu6.log
tail -3 gpurun_out/r02_pytest_gpu6.log
timeout 900 python tools/cosched.py --levels auto --tunes "graphs=1" --steps 50 > gpurun_out/r02_cosched_h2.log 2>&1
grep levels gpurun_out/r02_cosched_h2.log | cut -c1-450
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_bench_h2_$c.json 2> gpurun_out/r02_bench_h2_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r02_bench_h2_$c.json').read().strip().splitlines()[-1]);print('$c',round(d['value'],2),'Mpts/s',round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value'],2),d['detail']['representation']['level_modes'],'err',d['detail']['rel_err_vs_exact_200_rows'])" || tail -3 gpurun_out/r02_bench_h2_$c.err
done
