mkdir -p gpurun_out/c10
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_zz_bench_multirank.py > gpurun_out/c10/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c10/pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c10/$tag.json 2>gpurun_out/c10/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c10/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3), d.get('kv_cache',{}).get('blocks_released_per_step'))
"; }
for i in 1 2; do
BARGS="--config c2" run kv_fused_$i X=1
BARGS="--config c2" run kv_sep_$i DUCHESS_KV_FUSED=0
BARGS="--config c2nokv" run nokv_$i X=1
done
BARGS="--config c2 --shards 1" run kv_fused_s1 X=1
BARGS="--config c2 --shards 4" run kv_fused_s4 X=1
