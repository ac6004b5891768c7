#!/bin/bash
# after the K-chunked layer: config 2 with the layer as the overlap consumer, sanitizers over the layer
O=gpurun_out/r02b31; mkdir -p $O
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 > $O/bench_config2.json 2> $O/bench_config2.err
python - $O/bench_config2.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print("config2", d['value'], d['roofline']['frac'], d['e2e']['value'], d['parity']['exact'], o['consumer'][:40], o['hidden_frac_best'], o['hidden_frac_partitioned']['value'], o['consumer_roofline']['frac'])
PY
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_variants.py >> $O/sanitizer.txt 2>&1
done
grep -E "===|SUMMARY|ok$" $O/sanitizer.txt
