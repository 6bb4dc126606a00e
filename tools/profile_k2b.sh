#!/bin/bash
# ncu --set full captures of the barrier-free round kernel and advance kernel at C2, cold caches (run under gpurun).
mkdir -p gpurun_out
TAG=${1:-r01f}
for k in round_kernel advance_kernel; do
ncu --set full --cache-control none --clock-control none --import-source on -k regex:$k -s 5 -c 1 \
    -o gpurun_out/${k}_${TAG} -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/${k}_${TAG}.log 2>&1
done
ncu --set full --cache-control none --clock-control none --import-source on -k regex:decide_kernel -s 1 -c 1 \
    -o gpurun_out/decide_kernel_${TAG} -f python bench.py --steps 6 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/decide_${TAG}.log 2>&1
ls gpurun_out | grep $TAG
