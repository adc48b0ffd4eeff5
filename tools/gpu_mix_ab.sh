A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eval or full_moves or non_power" > gpurun_out/mx_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/mx_pytest.log
for wl in C2 C1 C4; do for mode in mixed homogeneous; do for r in 1 2; do
  echo "A $(PIPETTE_LIB=$A python tools/eval_probe.py $mode $wl)"
  echo "B $(python tools/eval_probe.py $mode $wl)"
done; done; done > gpurun_out/mx_ab.log 2>&1
echo "A C4 $(PIPETTE_LIB=$A python tools/search_probe.py C4 - - full)" >> gpurun_out/mx_ab.log 2>&1
echo "B C4 $(python tools/search_probe.py C4 - - full)" >> gpurun_out/mx_ab.log 2>&1
