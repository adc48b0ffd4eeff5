mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eval" > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
timeout 900 bash tools/ab_eval.sh > gpurun_out/e_ab.log 2>&1
