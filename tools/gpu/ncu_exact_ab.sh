#!/bin/bash
# ncu --set full of the exact-sum kernels of two library builds (A/B), same cases.
# Usage: bash tools/gpu/ncu_exact_ab.sh <a.so> <b.so> dtype:wl ...
set -u
mkdir -p gpurun_out
a=$1; b=$2; shift 2
for lib in "$a" "$b"; do
  tag=$(basename $(dirname $lib))
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rd_exact -o gpurun_out/prof_exact_$tag python tools/profile_lib.py $lib "$@" > gpurun_out/ncu_exact_$tag.log 2>&1; echo "ncu $tag=$?"
done
