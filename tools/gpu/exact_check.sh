mkdir -p gpurun_out; python -m paper_1710_07358_b200.build > /dev/null
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x --timeout 900 > gpurun_out/x3_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/x3_pytest.log
timeout 300 python tools/sweep.py exact --out gpurun_out/x3_exact.json > gpurun_out/x3_exact.log 2>&1; echo sweep=$?
python -c "
import json; d=json.load(open('gpurun_out/x3_exact.json'))
for r in d['result']:
  if r['op']=='sum_exact': print(r['dtype'], r['workload'], r['op'], round(r['gbps_med']), round(r.get('gbps_stream',0)), r['regs'], r['ctas_per_sm'])
"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rd_exact_kernel -o gpurun_out/x3_prof_exact python tools/profile_ops.py exact > gpurun_out/x3_ncu.log 2>&1; echo ncu=$?
