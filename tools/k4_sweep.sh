#!/bin/bash
# K4 (lr_grad) stage-size / register-keep sweep at C5 (run under gpurun).
mkdir -p gpurun_out/k4
for cfg in "32768 -1" "65536 -1" "65536 0" "131072 0" "32768 0" "16384 -1"; do
  set -- $cfg
  DUCHESS_K4_STAGE=$1 DUCHESS_K4_KEEP=$2 timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/k4/c5_$1_$2.json 2>/dev/null
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/k4/c5_$1_$2.json') if l.startswith('{')][-1])
print('stage $1 keep $2', round(d['value']/1e6,1), 'M rows/s', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])
"
done
