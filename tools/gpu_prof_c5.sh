mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_chains -c 1 -o gpurun_out/c5b_sa python tools/search_probe.py C5 4096 1000 > gpurun_out/c5_ncu.log 2>&1
