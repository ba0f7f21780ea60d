#!/bin/bash
# Fair A/B of two library builds on the exact sum: ABBA-ordered timing rounds per
# workload (optionally soaked), then ncu --set full of both on the same cases.
# Usage: bash tools/gpu/exact_ab_fair.sh <a.so> <b.so>
set -u
mkdir -p gpurun_out
a=$1; b=$2
for wl in u01 normalish wide; do
  AB_ROUNDS=4 AB_WORKLOAD=$wl AB_PAIRS=float32:sum_exact,float64:sum_exact timeout 600 python tools/ab_lib.py $a $b | sed "s/^{/{\"wl\": \"$wl\", /" >> gpurun_out/ab_fair.jsonl
done
bash tools/gpu/ncu_exact_ab.sh $a $b float32:u01 float64:u01 float64:normalish float32:wide float64:wide
