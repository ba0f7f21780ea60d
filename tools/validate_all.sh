#!/bin/bash
# Full round validation on one B200 (used under gpurun): GPU tests (incl. IPC / CLI), smoke,
# sanitizers (opt-in), bench (both arms), ncu launch list + full capture of the timed kernel.
set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1500 --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu=$?"
tail -1 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
# compute-sanitizer is closed on the GPU pool (runs under it left GPUs needing a reset):
# RD_VALIDATE_SANITIZE=1 runs the four tools where it is allowed
if [ -n "${RD_VALIDATE_SANITIZE:-}" ]; then
  for t in memcheck synccheck initcheck racecheck; do
    timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitize_$t.log 2>&1; echo "$t=$?"
  done
fi
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "bench_ref=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_default.csv python bench.py --steps 20 --warmup 3 --no-cpu > /dev/null 2>&1; echo "ncu_launches=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rd_bulk_kernel -s 5 -c 1 -o gpurun_out/prof_bulk_f32sum_final python bench.py --profile --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu_full=$?"
if [ -n "${RD_VALIDATE_REPORTS:-}" ]; then   # the measurement reports too (~8 min more)
  timeout 1500 python tools/c3_report.py --out gpurun_out/c3 > gpurun_out/c3.log 2>&1; echo "c3=$?"; tail -1 gpurun_out/c3.log
  timeout 900 python tools/sweep.py ops --log2n 28 --out gpurun_out/ops.json > /dev/null 2>&1; echo "ops=$?"
  timeout 300 python tools/sweep.py exact --out gpurun_out/exact.json > /dev/null 2>&1; echo "exact=$?"
fi
