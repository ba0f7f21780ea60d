#!/bin/bash
# Fair A/B of two library builds on the exact sum: the exact-sum GPU tests on the
# product build, ABBA-ordered timing rounds per workload, then (NCU=1) ncu --set full
# of both on the same cases.   Usage: bash tools/gpu/exact_ab_fair.sh <a.so> <b.so>
set -u
mkdir -p gpurun_out
a=$1; b=$2
timeout 1500 python -m pytest tests/test_gpu_exact.py -q -x --timeout 1200 > gpurun_out/pytest_exact.log 2>&1; echo "pytest=$?"; tail -1 gpurun_out/pytest_exact.log
for wl in ${AB_WLS:-u01 normalish wide wide_full}; do
  AB_ROUNDS=${AB_ROUNDS:-4} AB_WORKLOAD=$wl AB_PAIRS=float32:sum_exact,float64:sum_exact timeout 600 python tools/ab_lib.py $a $b | sed "s/^{/{\"wl\": \"$wl\", /" >> gpurun_out/ab_fair.jsonl
done
if [ -n "${NCU:-}" ]; then
  bash tools/gpu/ncu_exact_ab.sh $a $b float32:u01 float64:u01 float64:normalish float32:wide float64:wide float32:wide_full float64:wide_full
fi
