export PATH=/usr/local/cuda/bin:$PATH
for c in c5 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/r02_bench_half_$c.json 2> gpurun_out/r02_bench_half_$c.err
  python -c "import json;d=json.loads(open('gpurun_out/r02_bench_half_$c.json').read().strip().splitlines()[-1]);print('$c',round(d['value'],2),'Mpts/s',round(d['ms_per_step'],3),'ms e2e',round(d['e2e']['value'],2),d['detail']['representation']['level_modes'],'build',d['detail']['aca_build_s'],'err',d['detail']['rel_err_vs_exact_200_rows'])" || tail -3 gpurun_out/r02_bench_half_$c.err
done
