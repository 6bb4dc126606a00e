#!/bin/bash
# Run on the GPU box (gpurun): launch list of a short bench + one full ncu
# capture of the dominant kernel. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_fast -s 8 -c 1 \
    -o gpurun_out/k1_${TAG} -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/k1_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:decide -s 8 -c 1 \
    -o gpurun_out/decide_${TAG} -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/decide_ncu_${TAG}.log 2>&1
ls -la gpurun_out
