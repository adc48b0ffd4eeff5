mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --workload C5 --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
