#!/bin/bash
# ncu --set full captures of the K2 kernels (advance / decide) and K1 variants inside the C2 bench (run under gpurun).
mkdir -p gpurun_out
TAG=${1:-r01c}
for k in advance decide score_tma score_fast; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 \
    -o gpurun_out/${k}_${TAG} -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 --k1 ${K1:-list} > gpurun_out/${k}_${TAG}.log 2>&1
done
K1=ldg ncu --set full --clock-control none --import-source on -k regex:score_fast -s 6 -c 1 \
    -o gpurun_out/score_fast_${TAG} -f python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 2 --k1 ldg > gpurun_out/score_fast_${TAG}.log 2>&1
ls gpurun_out
