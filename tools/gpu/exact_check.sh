# exact-sum check on one B200: GPU parity tests, the workload sweep, an ncu capture of the fast path
mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
P=${1:-x}
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x --timeout 900 > gpurun_out/${P}_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/${P}_pytest.log
timeout 300 python tools/sweep.py exact --out gpurun_out/${P}_exact.json > gpurun_out/${P}_exact.log 2>&1; echo sweep=$?
python -c "
import json; d=json.load(open('gpurun_out/${P}_exact.json'))
for r in d['result']: print(r['dtype'], r['workload'], r['op'], r['variant'], round(r['gbps_med']), round(r.get('gbps_stream',0)), r['regs'], r['ctas_per_sm'])
"
if [ -n "$2" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rd_exact -o gpurun_out/${P}_prof_exact python tools/profile_ops.py exact > gpurun_out/${P}_ncu.log 2>&1; echo ncu=$?
fi
