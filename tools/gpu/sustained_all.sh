# bench-style SUSTAINED rate (1 s clock soak + 200 back-to-back steps) for every
# (dtype, op) of the north star, plus the extra ops, at 2^28
mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
for dt in int32 uint32 int64 float32 float64; do
  for op in sum prod min max and or xor argmin argmax sum_compensated sum_exact; do
    case "$dt:$op" in float*:and|float*:or|float*:xor) continue;; esac
    timeout 300 python bench.py --dtype $dt --op $op --steps 200 --warmup 3 --no-cpu --no-c5 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); rp=d['roofline'].get('read_probe') or {}; print(json.dumps({'dtype': '$dt', 'op': '$op', 'gbps': d['value'], 'probe_gbs': rp.get('value'), 'pct_probe': round(100*d['value']/rp['value'],2) if rp else None, 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons']}))"
  done
done > gpurun_out/sustained_all.jsonl
