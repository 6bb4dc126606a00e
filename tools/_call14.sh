mkdir -p gpurun_out/c14
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_zz_bench_multirank.py > gpurun_out/c14/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c14/pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c14/$tag.json 2>gpurun_out/c14/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c14/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3), d['counters'])
" || tail -3 gpurun_out/c14/$tag.err; }
for c in c2 c2nokv c3 c3t1; do
BARGS="--config $c" run ${c}_il DUCHESS_INTERLEAVE=1
BARGS="--config $c" run ${c}_ov DUCHESS_INTERLEAVE=0
done
BARGS="--config c2 --shards 3" run c2_il_s3 DUCHESS_INTERLEAVE=1
BARGS="--config c2 --shards 4" run c2_il_s4 DUCHESS_INTERLEAVE=1
