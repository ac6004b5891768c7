#!/bin/bash
# gathers at the maximum shared-memory carveout, sampler kernels at the driver's: default bench + overlap, cache mode
O=gpurun_out/r02b29; mkdir -p $O
timeout 900 python bench.py --no-baselines --timeline $O/overlap_timeline.json > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --cache-frac 0.2 --steps 20 --warmup 5 --no-baselines --no-overlap > $O/bench_cache20.json 2> $O/bench_cache20.err
python - $O <<'PY'
import json, sys
d=json.loads(open(sys.argv[1] + "/bench.json").read().splitlines()[-1]); o=d['overlap']
print("value", d['value'], "gather", d['roofline']['achieved'], "frac", d['roofline']['frac'], "e2e", d['e2e']['value'], "sample_p50", d['latency_ms']['fetch']['sample_p50'])
print(o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], "strict", o['hidden_frac_best'], "part", o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'])
c=json.loads(open(sys.argv[1] + "/bench_cache20.json").read().splitlines()[-1])
print("cache20", c['value'], c['latency_ms']['fetch']['sample_p50'])
PY
