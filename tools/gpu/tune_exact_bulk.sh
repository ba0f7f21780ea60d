# exact-sum bulk variant: consumer warps x expansions (RD_TUNE_EXACT_BULK="CW,E")
mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
P=${1:-xb}
for c in 16,2 16,1 24,2 24,1 8,2; do
  RD_TUNE_EXACT_BULK=$c timeout 300 python tools/tune_exact.py --variant bulk
done > gpurun_out/${P}_tune_exact_bulk.jsonl 2> gpurun_out/${P}_tune_exact_bulk.err
python - "$P" <<'PY'
import json, sys
for l in open(f"gpurun_out/{sys.argv[1]}_tune_exact_bulk.jsonl"):
    r = json.loads(l)
    print(r["cfg"], r["dtype"], r["workload"], round(r["gbps_med"]), round(r.get("gbps_stream", 0)), r["regs"])
PY
