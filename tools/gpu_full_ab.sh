A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "full_moves or non_power or byte_counts" > gpurun_out/fm_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fm_pytest.log
for wl in ${WLS:-C2 C3 C1}; do
  echo "A $wl $(PIPETTE_LIB=$A python tools/search_probe.py $wl - - full)"
  echo "B $wl $(python tools/search_probe.py $wl - - full)"
done > gpurun_out/fm_ab.log 2>&1
