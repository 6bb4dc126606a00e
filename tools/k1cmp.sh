# K1 last-token (T = 1) kernels side by side: register pipeline (mode 1) vs
# bulk-copy slots (mode 2); C3-T1 bench lines; optional ncu capture.
for m in 1 2; do DUCHESS_K1_ROWS=$m python tools/k1_short.py 0 1 4 5 > gpurun_out/k1short_m$m.txt 2>&1; cat gpurun_out/k1short_m$m.txt; done
if [ -n "$K1_BENCH" ]; then
  for m in 1 2; do DUCHESS_K1_ROWS=$m timeout 300 python bench.py --config c3t1 --steps 40 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/c3t1_m$m.json 2> gpurun_out/c3t1_m$m.err
  python -c "import json;d=json.load(open('gpurun_out/c3t1_m$m.json'));print('c3t1 mode $m', d['value'], d['roofline']['frac'], d['roofline'].get('vs_read_stream'))"; done
fi
timeout 600 python -m pytest tests/test_gpu_score.py tests/test_gpu_serving.py -x -q -p no:cacheprovider 2>&1 | tail -1
if [ -n "$K1_NCU" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:score_rows -s 5 -c 1 \
      -o gpurun_out/k1rows_bulk -f python tools/k1_short.py 0 > gpurun_out/k1rows_ncu.log 2>&1
  tail -1 gpurun_out/k1rows_ncu.log
fi
