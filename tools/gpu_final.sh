# Round-end GPU pass: parity suite, per-workload search/eval probes, bench, launch list, ncu.
mkdir -p gpurun_out
T=${TAG:-g}
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for wl in C1 C2 C3 C4 C5; do python tools/search_probe.py $wl; done > gpurun_out/${T}_search.log 2>&1
for wl in C2 C3 C4 C5; do python tools/search_probe.py $wl - - full; done > gpurun_out/${T}_search_full.log 2>&1
for wl in C1 C2 C3 C4 C5; do for m in homogeneous mixed; do python tools/eval_probe.py $m $wl; done; done > gpurun_out/${T}_eval.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/${T}_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sa_chains -c 1 -o gpurun_out/${T}_sa python tools/search_probe.py C2 > gpurun_out/${T}_ncu_sa.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_eval_stream -c 1 -o gpurun_out/${T}_eval python tools/eval_probe.py homogeneous C2 > gpurun_out/${T}_ncu_eval.log 2>&1
