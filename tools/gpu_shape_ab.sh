# A/B of K3 block shapes (lib/ab variants from tools/ab_variants.sh) on C1/C2, alternating.
mkdir -p gpurun_out
L=paper_2405_18093_b200/lib
for rep in 1 2 3; do for wl in C2 C1; do for v in main ${VARIANTS:-t128b4 t64b8 t64b6}; do
  lib=$L/libpipette.so; [ $v != main ] && lib=$L/ab/libpipette_$v.so
  echo "$v $(PIPETTE_LIB=$lib timeout 120 python tools/search_probe.py $wl 2>&1 | tail -1)"
done; done; done > gpurun_out/shape_ab.log 2>&1
for v in ${VARIANTS:-t128b4 t64b8 t64b6}; do
  PIPETTE_LIB=$L/ab/libpipette_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "search" > gpurun_out/shape_pytest_$v.log 2>&1; echo "rc=$?" >> gpurun_out/shape_pytest_$v.log
done
