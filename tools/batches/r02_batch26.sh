#!/bin/bash
# fetch-path kernels with the maximum shared-memory carveout (default now): parity, attribution, bench
O=gpurun_out/r02b26; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sage.py -q -x 2>&1 | tail -1
ATTRIB_KINDS=spin,gather,gather_primary timeout 300 python tools/explore/overlap_attrib.py --sms 64 --warps 1 | grep corunner | tee $O/attrib_64x1.jsonl
ATTRIB_KINDS=spin,gather,gather_primary timeout 300 python tools/explore/overlap_attrib.py --sms 24 --warps 2 | grep corunner | tee $O/attrib_24x2.jsonl
timeout 900 python bench.py --no-baselines --timeline $O/overlap_timeline.json > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print("value", d['value'], "gather", d['roofline']['achieved'], "frac", d['roofline']['frac'], "e2e", d['e2e']['value'])
print(o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], "strict", o['hidden_frac_best'], "part", o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'])
for r in o['sweep']:
    print(r.get('shape'), r.get('t_fetch_ms'), r.get('t_consumer_ms'), r.get('t_step_overlapped_ms'))
PY
