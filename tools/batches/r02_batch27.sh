#!/bin/bash
# overlap leg with a fifth sampler placement: its own high-priority stream on the whole GPU
O=gpurun_out/r02b27; mkdir -p $O
timeout 900 python bench.py --no-baselines --timeline $O/overlap_timeline.json > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print("value", d['value'], "gather", d['roofline']['achieved'], "frac", d['roofline']['frac'], "e2e", d['e2e']['value'])
print(o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], "strict", o['hidden_frac_best'], "part", o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'])
for r in o['sweep']:
    if 'shape' in r and r['shape'][4] == 'whole GPU': print(r.get('shape'), r.get('t_fetch_ms'), r.get('t_consumer_ms'), r.get('t_step_overlapped_ms'))
tl=o['timeline']
for st in tl['steps'][:5]:
    s,g,c=st['sample'],st['gather'],st['consume']
    print(st['step'], 'sample %.2f-%.2f' % tuple(s), 'gather %.2f-%.2f' % tuple(g), 'consume %.2f-%.2f (%.2f)' % (c[0], c[1], c[1]-c[0]))
PY
