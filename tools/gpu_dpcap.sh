# C5 search time vs the psum cache cap (PIPETTE_DP_CAP) of the BIG MODE 1 kernel.
mkdir -p gpurun_out
for cap in none 4 8 16 32; do
  if [ $cap = none ]; then echo "cap=$cap $(python tools/search_probe.py ${WL:-C5})";
  else echo "cap=$cap $(PIPETTE_DP_CAP=$cap python tools/search_probe.py ${WL:-C5})"; fi
done > gpurun_out/dpcap.log 2>&1
