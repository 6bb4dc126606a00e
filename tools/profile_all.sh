#!/bin/bash
# Round profile pass (run under gpurun, 1 GPU). Outputs in gpurun_out/prof_<tag>/;
# summarised into profiles/<tag>/ by tools/summarize_profiles.py <tag>.
TAG=${1:-r02}
D=gpurun_out/prof_$TAG
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $D/gpu.txt
# launch list of the default bench (C2: K1 + K2 + K3 per round and shard)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $D/launches_c2.csv python bench.py --config c2 --steps 8 --warmup 3 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/bench_c2_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_tma -s 2 -c 1 -o $D/k1_full -f python tools/k1_capture.py > $D/k1_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:score_rows -s 5 -c 1 -o $D/k1rows_full -f python tools/k1_short.py 0 > $D/k1rows_full.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:^round_kernel -s 40 -c 1 -o $D/round_full -f python bench.py --config c2 --steps 8 --warmup 3 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/round_full.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:kv_round_kernel -s 40 -c 1 -o $D/kv_full -f python bench.py --config c2 --steps 8 --warmup 3 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/kv_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fork_exec -s 2 -c 1 -o $D/k3_full -f python bench.py --config c4 --steps 3 --warmup 1 --no-cpu-baseline --no-gate > $D/k3_full.log 2>&1
DUCHESS_C5_ROWS=524288 ncu --set full --clock-control none --import-source on -k regex:lr_grad_ -s 2 -c 1 -o $D/k4_full -f python bench.py --config c5 --steps 3 --warmup 1 --no-cpu-baseline --no-gate > $D/k4_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:linear_kernel -s 2 -c 1 -o $D/mlp1_full -f python bench.py --config c3mlp --steps 3 --warmup 1 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/mlp1_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mlp_probe_tc -s 2 -c 1 -o $D/mlp2_full -f python bench.py --config c3mlp --steps 3 --warmup 1 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/mlp2_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:linear_kernel -s 4 -c 1 -o $D/tc_full -f python bench.py --config difficulty --steps 3 --warmup 1 --no-cpu-baseline > $D/tc_full.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"linear_kernel|row_normalize_bulk|head_reg" -s 20 -c 5 \
    --csv --log-file $D/launches_difficulty.csv python bench.py --config difficulty --steps 6 --warmup 3 --no-cpu-baseline > $D/bench_difficulty_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $D/launches_c3mlp.csv python bench.py --config c3mlp --steps 4 --warmup 2 --no-cpu-baseline --no-gate --e2e-steps 2 > $D/bench_c3mlp_under_ncu.log 2>&1
ls -la $D
