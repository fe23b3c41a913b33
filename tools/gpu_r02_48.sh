export PATH=/usr/local/cuda/bin:$PATH
nproc; lscpu | grep "Model name"
(time timeout 2400 python bench.py --impl reference --steps 3 --warmup 1) > gpurun_out/r02_bench_ref_cpu.json 2> gpurun_out/r02_bench_ref_cpu.err; echo "ref rc=$?"
cat gpurun_out/r02_bench_ref_cpu.json | cut -c1-1500; tail -5 gpurun_out/r02_bench_ref_cpu.err
