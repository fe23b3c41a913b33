export PATH=/usr/local/cuda/bin:$PATH
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu4.log
tail -3 gpurun_out/r02_pytest_gpu4.log
for c in c3 c4 c2 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_bench_half_$c.json 2> gpurun_out/r02_bench_half_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r02_bench_half_$c.json').read().strip().splitlines()[-1]);print('$c',round(d['value'],2),'Mpts/s',round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value'],2),d['detail']['representation']['level_modes'],'build',d['detail']['aca_build_s'],'err',d['detail']['rel_err_vs_exact_200_rows'])"
done
