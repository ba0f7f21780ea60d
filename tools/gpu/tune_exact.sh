# exact-sum vector kernel shapes (RD_TUNE_EXACT="U,E,MINB": loads in flight,
# expansions, min CTAs/SM) -- only the configurations rd_inst_exact.cu compiles
mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
for c in 6,2,2 6,2,1 4,2,2 8,1,2 2,2,3; do
  RD_TUNE_EXACT=$c timeout 300 python tools/tune_exact.py
done > gpurun_out/x8_tune_exact.jsonl 2> gpurun_out/x8_tune_exact.err
python - <<'PY'
import json
for l in open("gpurun_out/x8_tune_exact.jsonl"):
    r = json.loads(l)
    print(r["cfg"], r["dtype"], r["workload"], round(r["gbps_med"]), r["regs"], r["ctas_per_sm"])
PY
