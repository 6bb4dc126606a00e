mkdir -p gpurun_out/c13
timeout 900 python -m pytest tests/test_gpu_kvcache.py -x -q -p no:cacheprovider > gpurun_out/c13/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c13/pytest.log
python tools/trace_round.py 128 c2 kv > gpurun_out/c13/trace_kv.txt 2>&1; tail -4 gpurun_out/c13/trace_kv.txt
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c13/$tag.json 2>gpurun_out/c13/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c13/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3))
"; }
BARGS="--config c2" run after DUCHESS_KV_TAILS=after
BARGS="--config c2" run overlap DUCHESS_KV_TAILS=overlap
BARGS="--config c2" run sep DUCHESS_KV_FUSED=0
BARGS="--config c2nokv" run nokv X=1
