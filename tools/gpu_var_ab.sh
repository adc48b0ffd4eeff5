# Same-box A/B of lib/ab variants (VARIANTS) against the in-tree lib: SA search on C2/C3,
# alternating, then the SA parity tests on each variant.
mkdir -p gpurun_out
L=paper_2405_18093_b200/lib
for rep in 1 2 3; do for wl in ${WLS:-C2 C3}; do for v in main $VARIANTS; do
  lib=$L/libpipette.so; [ $v != main ] && lib=$L/ab/libpipette_$v.so
  echo "$v $(PIPETTE_LIB=$lib timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
done; done; done > gpurun_out/var_ab.log 2>&1
for v in $VARIANTS; do
  PIPETTE_LIB=$L/ab/libpipette_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "search" > gpurun_out/var_pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/var_pytest_$v.log
done
