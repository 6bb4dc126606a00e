mkdir -p gpurun_out/c15
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_zz_bench_multirank.py > gpurun_out/c15/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c15/pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c15/$tag.json 2>gpurun_out/c15/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c15/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3))
" || tail -3 gpurun_out/c15/$tag.err; }
for i in 1 2; do
BARGS="--config c2" run lead_$i DUCHESS_KV_MODE=lead
BARGS="--config c2" run overlap_$i DUCHESS_KV_MODE=overlap
BARGS="--config c2" run fused_$i DUCHESS_KV_MODE=fused
BARGS="--config c2nokv" run nokv_$i X=1
done
BARGS="--config c2 --shards 1" run lead_s1 DUCHESS_KV_MODE=lead
BARGS="--config c2 --shards 4" run lead_s4 DUCHESS_KV_MODE=lead
