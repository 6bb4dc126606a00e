mkdir -p gpurun_out/c7
for i in 1 2 3; do for c in c2 c2nokv; do timeout 300 python bench.py --config $c --no-cpu-baseline --e2e-steps 2 > gpurun_out/c7/b_${c}_$i.json 2>/dev/null; python -c "
import json
d=json.loads([l for l in open('gpurun_out/c7/b_${c}_$i.json') if l.startswith('{')][-1])
print('$c', $i, round(d['value']/1e6,2), round(d['ms_per_step']*1e3,1), round(d['roofline']['vs_read_stream']['frac'],3), round(d['roofline']['vs_read_stream']['peak']))
"; done; done
