mkdir -p gpurun_out/c11
python tools/trace_round.py 128 c2 kv > gpurun_out/c11/trace_kv.txt 2>&1
python tools/trace_round.py 128 c2nokv > gpurun_out/c11/trace_nokv.txt 2>&1
cat gpurun_out/c11/*.txt
