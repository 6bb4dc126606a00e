#!/bin/bash
# K1 variants at C2 inside the full bench step
for cfg in "1 16384" "1 32768" "2 16384" "2 8192" "3 8192" "4 8192"; do
  set -- $cfg
  DUCHESS_K1_CPS=$1 DUCHESS_K1_STAGE=$2 python bench.py --no-cpu-baseline --steps 100 --k1 list 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma cps=$1 stage=$2', round(d['value']/1e6,3), 'M/s step_us', round(d['ms_per_step']*1e3,1), 'k1_us', round(d['roofline']['k1_us_per_launch'],1), 'frac', round(d['roofline']['frac'],3))"
done
for cfg in "2 128" "1 256" "4 128"; do
  set -- $cfg
  python bench.py --no-cpu-baseline --steps 100 --k1 ldg --nsplit $1 --threads $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ldg ns=$1 nt=$2', round(d['value']/1e6,3), 'M/s step_us', round(d['ms_per_step']*1e3,1), 'k1_us', round(d['roofline']['k1_us_per_launch'],1), 'frac', round(d['roofline']['frac'],3))"
done
