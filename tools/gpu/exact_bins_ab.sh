#!/bin/bash
# A/B of the exact sum's fallback (bins) against a baseline library build, per workload;
# exact-sum GPU tests first. Usage: bash tools/gpu/exact_bins_ab.sh [other.so ...]
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_exact.py -q -x --timeout 1200 > gpurun_out/pytest_exact_bins.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_exact_bins.log
for wl in u01 normalish wide wide_full; do
  AB_WORKLOAD=$wl AB_PAIRS=float32:sum_exact,float64:sum_exact timeout 600 python tools/ab_lib.py build/ab/base/libb200reduce.so paper_1710_07358_b200/libb200reduce.so "$@" | sed "s/^{/{\"wl\": \"$wl\", /" >> gpurun_out/ab_bins.jsonl
done
cat gpurun_out/ab_bins.jsonl
