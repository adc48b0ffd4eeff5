#!/usr/bin/env bash
# One driver for the GPU-side jobs of this repo, run on a B200 box through gpurun, e.g.
#   gpurun --timeout 1800 -- 'bash tools/gpu.sh parity'
#   gpurun --timeout 1800 -- 'bash tools/gpu.sh ab paper_2405_18093_b200/lib/ab/libpipette_HEAD.so C5 C4'
#   gpurun --timeout 1800 -- 'bash tools/gpu.sh profile k_sa_chains TAG python tools/search_probe.py C5 4096 1000'
#   gpurun --gpus 4 --timeout 3600 -- 'bash tools/gpu.sh scale C5 4'
# Outputs go to gpurun_out/ (scratch; copy what is judged into profiles/).
#   parity              full GPU test suite (tests -m gpu)
#   ab LIB_A WL...      alternating A/B of pipette_search: LIB_A (PIPETTE_LIB) vs the working
#                       tree's library, two reps per workload, + task profiles of B
#   profile RE TAG CMD  CMD once plainly (must exit 0), then ncu --set full on the first kernel
#                       matching RE, digested on the box (tools/ncu_digest.py) so only the
#                       digest travels back (a report is ~10-20 MB; gpurun_out/ is capped)
#   scale WL NMAX       bench.py strong scaling at N = 1, 2, 4, ... NMAX (torchrun for N > 1),
#                       then tests/test_gpu_multi.py
#   bench               the default bench line (what the driver runs at round end)
#   sanitize            tools/sanitize_suite.py plainly (compute-sanitizer is closed on this pool)
set -u
mkdir -p gpurun_out
cmd=${1:-parity}; shift || true
case "$cmd" in
  parity)
    timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log ;;
  ab)
    A=$1; shift
    for rep in 1 2; do for wl in "$@"; do
      echo "A $(PIPETTE_LIB=$A timeout 600 python tools/search_probe.py $wl 2>&1 | tail -1)"
      echo "B $(timeout 600 python tools/search_probe.py $wl 2>&1 | tail -1)"
    done; done > gpurun_out/ab.log 2>&1
    for wl in "$@"; do timeout 600 python tools/task_profile.py $wl > gpurun_out/tasks_$wl.log 2>&1; done ;;
  profile)
    RE=$1; TAG=$2; shift 2
    "$@" > gpurun_out/profile_${TAG}_plain.log 2>&1 && \
    timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$RE -c 1 -o /tmp/prof_$TAG "$@" \
      > gpurun_out/profile_${TAG}_ncu.log 2>&1 && \
    python tools/ncu_digest.py /tmp/prof_$TAG.ncu-rep > gpurun_out/profile_${TAG}_digest.txt 2>&1 ;;
  scale)
    WL=${1:-C5}; NMAX=${2:-4}
    nvidia-smi topo -m > gpurun_out/scale_topo.txt 2>&1
    timeout 900 python bench.py --workload $WL --steps 5 --warmup 3 --no-eval --no-cpu --no-extra \
      > gpurun_out/scale_${WL}_n1.json 2> gpurun_out/scale_${WL}_n1.err
    N=2
    while [ $N -le $NMAX ]; do
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29517 bench.py --workload $WL --gpus $N --steps 5 --warmup 3 --no-eval --no-extra \
        > gpurun_out/scale_${WL}_n$N.json 2> gpurun_out/scale_${WL}_n$N.err
      N=$((N * 2))
    done
    timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/scale_multi.log 2>&1 ;;
  bench)
    timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ;;
  sanitize)
    timeout 1200 python tools/sanitize_suite.py > gpurun_out/sanitize.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize.log ;;
  *) echo "unknown command $cmd"; exit 2 ;;
esac
