mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_chains -c 1 -o gpurun_out/c5_sa python tools/search_probe.py C5 4096 1000 > gpurun_out/c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sa_chains -c 1 -o gpurun_out/c4_sa python tools/search_probe.py C4 1024 2000 > gpurun_out/c4_ncu.log 2>&1
