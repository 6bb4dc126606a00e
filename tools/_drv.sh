mkdir -p gpurun_out/drv2
( time timeout 1500 python3 bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/drv2/bench.json 2> gpurun_out/drv2/bench.err
( time timeout 1500 python3 bench.py ) > gpurun_out/drv2/bench_k200.json 2> gpurun_out/drv2/bench_k200.err
