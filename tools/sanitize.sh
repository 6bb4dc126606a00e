#!/bin/bash
# compute-sanitizer pass over the GPU parity tests (run under gpurun, 1 GPU).
# Outputs in gpurun_out/san/.
mkdir -p gpurun_out/san

T2="tests/test_gpu_score.py tests/test_gpu_step.py tests/test_gpu_kvfork_train.py tests/test_gpu_mlp_tc.py tests/test_gpu_difficulty.py tests/test_gpu_facade.py tests/test_simulation.py"
for tool in memcheck racecheck synccheck; do
  compute-sanitizer --tool $tool --log-file gpurun_out/san/$tool.log \
      python -m pytest tests/test_gpu_edge.py tests/test_gpu_engine.py -q -x -k "not widest" > gpurun_out/san/$tool.out 2>&1
done
compute-sanitizer --tool memcheck --log-file gpurun_out/san/memcheck_all.log \
    python -m pytest $T2 -m gpu -q -x > gpurun_out/san/memcheck_all.out 2>&1
compute-sanitizer --tool synccheck --log-file gpurun_out/san/synccheck_all.log \
    python -m pytest tests/test_gpu_score.py tests/test_gpu_step.py tests/test_gpu_kvfork_train.py \
    tests/test_gpu_mlp_tc.py tests/test_gpu_difficulty.py -q -x > gpurun_out/san/synccheck_all.out 2>&1
tail -n 2 gpurun_out/san/*.log
