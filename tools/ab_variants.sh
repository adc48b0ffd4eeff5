#!/bin/bash
# Build libpipette.so variants of the working tree with extra nvcc flags, in parallel, into
# paper_2405_18093_b200/lib/ab/libpipette_<name>.so.   usage: ab_variants.sh name="-D.. -D.." ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/paper_2405_18093_b200/lib/ab"
pids=()
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  d=/tmp/pipette_var_$name; rm -rf "$d"; mkdir -p "$d"
  cp -r "$ROOT/paper_2405_18093_b200" "$ROOT/include" "$d/"
  rm -rf "$d/paper_2405_18093_b200/lib"
  ( cd "$d" && PIPETTE_NVCC_EXTRA="$flags" python -m paper_2405_18093_b200.build --force > build.log 2>&1 &&
    cp paper_2405_18093_b200/lib/libpipette.so "$ROOT/paper_2405_18093_b200/lib/ab/libpipette_$name.so" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
ls -la "$ROOT/paper_2405_18093_b200/lib/ab"
