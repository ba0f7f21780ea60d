mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
for c in 4,2,1 6,2,1 2,2,3 4,2,2; do
  RD_TUNE_EXACT=$c timeout 300 python tools/tune_exact.py
done > gpurun_out/x8_tune_exact.jsonl 2> gpurun_out/x8_tune_exact.err
python - <<'PY'
import json
for l in open("gpurun_out/x8_tune_exact.jsonl"):
    r = json.loads(l)
    print(r["cfg"], r["dtype"], r["workload"], round(r["gbps_med"]), r["regs"], r["ctas_per_sm"])
PY
