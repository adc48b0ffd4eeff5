# A/B of the SA search (baseline lib $1 vs the working tree's lib) + SA parity tests.
A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "search or full_moves or non_power" > gpurun_out/sa_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/sa_pytest.log
for wl in ${WLS:-C2 C3 C4}; do for rep in 1 2; do
  echo "A $wl $(PIPETTE_LIB=$A python tools/search_probe.py $wl)"
  echo "B $wl $(python tools/search_probe.py $wl)"
done; done > gpurun_out/sa_ab.log 2>&1
