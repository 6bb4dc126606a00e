#!/bin/bash
# compute-sanitizer pass over the GPU parity tests (run under gpurun, 1 GPU).
# Outputs in gpurun_out/san/; summarised into profiles/<round>/sanitizer/.
mkdir -p gpurun_out/san

# K2 (split / round kernels), K3 in the round (both launch modes, incl. the
# serving loop whose scorer streams beside K3), K1 list / rows kernels
CORE="tests/test_gpu_edge.py tests/test_gpu_engine.py tests/test_gpu_kvcache.py"
for tool in memcheck racecheck synccheck; do
  timeout 2400 compute-sanitizer --tool $tool --log-file gpurun_out/san/$tool.log \
      python -m pytest $CORE -q -x -k "not widest" -p no:cacheprovider > gpurun_out/san/$tool.out 2>&1
done
# everything else with a GPU kernel (memcheck; synccheck for the kernels with barriers)
T2="tests/test_gpu_score.py tests/test_gpu_kvfork_train.py tests/test_gpu_mlp_tc.py tests/test_gpu_mlp_paper.py
    tests/test_gpu_difficulty.py tests/test_gpu_facade.py tests/test_gpu_upload.py tests/test_simulation.py"
timeout 2400 compute-sanitizer --tool memcheck --log-file gpurun_out/san/memcheck_all.log \
    python -m pytest $T2 -m gpu -q -x -p no:cacheprovider > gpurun_out/san/memcheck_all.out 2>&1
timeout 2400 compute-sanitizer --tool synccheck --log-file gpurun_out/san/synccheck_all.log \
    python -m pytest tests/test_gpu_score.py tests/test_gpu_kvfork_train.py tests/test_gpu_mlp_tc.py \
    tests/test_gpu_mlp_paper.py tests/test_gpu_difficulty.py -q -x -p no:cacheprovider \
    > gpurun_out/san/synccheck_all.out 2>&1
tail -n 2 gpurun_out/san/*.log gpurun_out/san/*.out
