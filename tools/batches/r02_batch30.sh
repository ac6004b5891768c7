#!/bin/bash
# overlap leg with a 3-slot ring (fetch two minibatches ahead) vs the ping-pong pair
O=gpurun_out/r02b30; mkdir -p $O
for sl in 3 2; do
  timeout 900 python bench.py --no-baselines --overlap-slots $sl --timeline $O/overlap_timeline_s$sl.json > $O/bench_s$sl.json 2> $O/bench_s$sl.err
  python - $O/bench_s$sl.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print(sys.argv[1], o['t_fetch_ms'], o['t_consumer_ms'], "strict", o['hidden_frac_best'], "part", o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'])
for st in o['timeline']['steps'][:5]:
    s,g,c=st['sample'],st['gather'],st['consume']
    print(st['step'], 'sample %.2f-%.2f' % tuple(s), 'gather %.2f-%.2f (%.2f)' % (g[0],g[1],g[1]-g[0]), 'consume %.2f-%.2f (%.2f)' % (c[0], c[1], c[1]-c[0]))
PY
done
