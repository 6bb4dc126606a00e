#!/bin/bash
# K3 (fork_exec, C4) tail-copy unroll sweep (run under gpurun).
mkdir -p gpurun_out/k3
for u in 4 8 16 4 8 16; do
  DUCHESS_K3_UNROLL=$u timeout 300 python bench.py --config c4 --no-cpu-baseline > gpurun_out/k3/c4_$u.json 2>/dev/null
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/k3/c4_$u.json') if l.startswith('{')][-1])
print('unroll $u', round(d['value']/1e6,1), 'M forks/s', round(d['roofline']['frac'],3))
"
done
