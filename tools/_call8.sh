mkdir -p gpurun_out/c8
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c8/$tag.json 2>gpurun_out/c8/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c8/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3))
"; }
BARGS="--config c2" run kv_ovl X=1
BARGS="--config c2" run kv_ser DUCHESS_KV_OVERLAP=0
BARGS="--config c2nokv" run nokv X=1
BARGS="--config c2 --shards 1" run kv_ovl_s1 X=1
BARGS="--config c2 --shards 1" run kv_ser_s1 DUCHESS_KV_OVERLAP=0
BARGS="--config c2nokv --shards 1" run nokv_s1 X=1
BARGS="--config c2 --shards 4" run kv_ovl_s4 X=1
BARGS="--config c2nokv --shards 4" run nokv_s4 X=1
