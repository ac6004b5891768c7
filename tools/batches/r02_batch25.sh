#!/bin/bash
# overlap leg with the layer launched persistent (2 CTAs per SM, one launch per step) vs short launches
O=gpurun_out/r02b25; mkdir -p $O
for cps in 2 0; do
  timeout 900 python bench.py --no-baselines --consumer-ctas-per-sm $cps > $O/bench_cps$cps.json 2> $O/bench_cps$cps.err
  python - $O/bench_cps$cps.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print(sys.argv[1], d['value'], o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], o['hidden_frac_best'], o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'])
PY
done
