#!/bin/bash
# K4 (lr_grad) variant sweep at C5 (run under gpurun): stage bytes, keep mode
# (1 = one warp set keeping the stage in registers, 0 = re-read) and the
# split dot / grad warp sets (DUCHESS_K4_SPLIT=1).
mkdir -p gpurun_out/k4
for cfg in "32768 -1 0" "32768 -1 1" "65536 -1 1" "16384 -1 1" "131072 -1 1"; do
  set -- $cfg
  tag=$1_$2_$3
  DUCHESS_K4_STAGE=$1 DUCHESS_K4_KEEP=$2 DUCHESS_K4_SPLIT=$3 timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/k4/c5_$tag.json 2>/dev/null
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/k4/c5_$tag.json') if l.startswith('{')][-1])
print('stage $1 keep $2 split $3', round(d['value']/1e6,1), 'M rows/s', round(d['roofline']['frac'],3), d['roofline'].get('vs_read_stream'), d['clocks']['sm_mhz'])
"
done
