#!/bin/bash
# Sweep of the bulk chunk-schedule knobs (rd_api.cu env_u64): bench.py --profile value per setting.
for cfg in ${TUNE_CFGS:-"12 4 2" "12 16 1" "12 32 1" "16 16 1" "12 8 1" "18 16 1" "12 24 1" "8 16 1"}; do
  set -- $cfg
  for rep in 1 2; do
    v=$(RD_TUNE_HEAD_PER_SM=$1 RD_TUNE_TAIL_PER_SM=$2 RD_TUNE_TAIL_STAGES=$3 timeout 120 python bench.py --profile --steps 200 --warmup 10 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])")
    echo "head=$1 tail=$2 tailstages=$3 rep=$rep value=$v"
  done
done
