mkdir -p gpurun_out/c6
( time timeout 1500 python bench.py ) > gpurun_out/c6/bench_default.json 2> gpurun_out/c6/bench_default.err
timeout 900 python -m pytest tests/test_gpu_zz_bench_multirank.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > gpurun_out/c6/pytest_mr.log 2>&1; echo mr rc=$?
ncu --set full --cache-control none --clock-control none --import-source on -k regex:^round_kernel -s 40 -c 1 -o gpurun_out/c6/round_full -f python bench.py --config c2 --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c6/round_full.log 2>&1
