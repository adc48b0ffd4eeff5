A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eval" > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
for wl in C4 C5; do for mode in homogeneous mixed; do
  echo "A $(PIPETTE_LIB=$A python tools/eval_probe.py $mode $wl)"
  echo "B $(python tools/eval_probe.py $mode $wl)"
done; done > gpurun_out/e_ab.log 2>&1
