set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/d_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d_pytest.log
timeout 600 python bench.py > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload C5 --no-cpu --no-e2e --steps 3 --warmup 3 > gpurun_out/d_bench_c5.json 2> gpurun_out/d_bench_c5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/d_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/d_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_chains -c 1 -o gpurun_out/d_sa python tools/search_probe.py C2 > gpurun_out/d_ncu_sa.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_stream -c 1 -o gpurun_out/d_eval python tools/eval_probe.py homogeneous C2 > gpurun_out/d_ncu_eval.log 2>&1
ls gpurun_out
