# Same-box A/B of the working tree's lib (B) against lib/ab/libpipette_HEAD.so (A): full GPU
# parity suite on B, then SA search (C2, C1, C3) and eval stream (C2, C1) alternating.
A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_pytest.log
for rep in 1 2 3; do for wl in C2 C3; do
  echo "A $(PIPETTE_LIB=$A timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
  echo "B $(timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
done; done > gpurun_out/ab_sa.log 2>&1
for rep in 1 2; do for wl in C2 C1; do for mode in homogeneous mixed; do
  echo "A $(PIPETTE_LIB=$A timeout 120 python tools/eval_probe.py $mode $wl 2>&1 | tail -1)"
  echo "B $(timeout 120 python tools/eval_probe.py $mode $wl 2>&1 | tail -1)"
done; done; done > gpurun_out/ab_eval.log 2>&1
