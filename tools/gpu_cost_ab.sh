# Same-box A/B of the K3 task cost model: PIPETTE_COST_FIT=0 (A, the earlier estimate) vs the
# default fitted model (B), alternating; then the SA parity tests with the default.
mkdir -p gpurun_out
for rep in 1 2 3; do for wl in ${WLS:-C2 C3 C4 C5}; do
  echo "A $(PIPETTE_COST_FIT=0 timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
  echo "B $(timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
done; done > gpurun_out/cost_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "search or full_moves" > gpurun_out/cost_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/cost_pytest.log
