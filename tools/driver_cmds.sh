#!/bin/bash
# The driver's round-end bench commands on one GPU (run under gpurun): the
# 1-GPU line (K = 20, every config under `secondary`), the default K = 200
# line, and the reference arm.
mkdir -p gpurun_out/drv
( time timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/drv/bench.json 2> gpurun_out/drv/bench.err
( time timeout 1500 python3 bench.py ) > gpurun_out/drv/bench_k200.json 2> gpurun_out/drv/bench_k200.err
( time timeout 900 python3 bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/drv/reference.json 2> gpurun_out/drv/reference.err
