mkdir -p gpurun_out/c5
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_zz_bench_multirank.py > gpurun_out/c5/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c5/pytest.log
python tools/trace_round.py 128 > gpurun_out/c5/trace128.txt 2>&1
python tools/trace_round.py 8 c1 > gpurun_out/c5/trace_c1.txt 2>&1
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/c5/bench_$c.json 2> gpurun_out/c5/bench_$c.err; done
cat gpurun_out/c5/trace*.txt
