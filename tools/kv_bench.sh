# C2 serving step with and without K3 in the round (paged KV cache).
python_line() { python -c "
import json;d=json.load(open('$1'));print('$2', round(d['value']/1e6,2), 'M/s', round(d['ms_per_step']*1e3,1), 'us/step', d.get('kv_cache',{}).get('blocks_allocated_per_step'), d['e2e']['value'])"; }
for c in c2nokv c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_$c.json 2> gpurun_out/b_$c.err; python_line gpurun_out/b_$c.json $c; done
if [ -n "$KV_MODES" ]; then
for c in c2nokv c2; do timeout 300 python bench.py --config $c --shards 1 --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 2 > gpurun_out/b1_$c.json 2>/dev/null; python_line gpurun_out/b1_$c.json "$c shards=1"; done
fi
