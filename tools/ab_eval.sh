# A/B of the eval stream: baseline lib (argument 1) vs the working tree's lib, same box.
A=${1:-paper_2405_18093_b200/lib/ab/libpipette_HEAD.so}
for wl in C2 C3 C1; do for mode in homogeneous mixed; do
  for rep in 1 2; do
    echo "A $(PIPETTE_LIB=$A python tools/eval_probe.py $mode $wl)"
    echo "B $(python tools/eval_probe.py $mode $wl)"
  done
done; done
