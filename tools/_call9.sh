mkdir -p gpurun_out/c9
run() { tag=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --e2e-steps 2 --secondary none $BARGS > gpurun_out/c9/$tag.json 2>gpurun_out/c9/$tag.err; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c9/$tag.json') if l.startswith('{')][-1])
print('$tag', round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3))
"; }
BARGS="--config c2" run kv_cps1 DUCHESS_K1_CPS=1
BARGS="--config c2nokv" run nokv_cps1 DUCHESS_K1_CPS=1
BARGS="--config c2" run kv_cps2 DUCHESS_K1_CPS=2
BARGS="--config c2 --shards 4" run kv_cps1_s4 DUCHESS_K1_CPS=1
BARGS="--config c2nokv --shards 4" run nokv_cps1_s4 DUCHESS_K1_CPS=1
BARGS="--config c3" run c3_cps1 DUCHESS_K1_CPS=1
BARGS="--config c3" run c3_cps2 DUCHESS_K1_CPS=2
