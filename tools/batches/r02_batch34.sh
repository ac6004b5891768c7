#!/bin/bash
# final records for the layer (dynamic schedule + TMA stores): GPU suite, roofline, ncu --set full, sanitizers,
# the default bench line
O=gpurun_out/r02b34; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu > $O/gputest.txt 2>&1; tail -1 $O/gputest.txt
timeout 300 python tools/consumer_roofline.py > $O/consumer_roofline.jsonl 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sage_mean --launch-skip 5 --launch-count 1 \
    -o $O/ncu_sage python tools/consumer_roofline.py --iters 2 > $O/ncu_sage.log 2>&1
for tool in memcheck racecheck synccheck; do
  echo "=== $tool" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_variants.py >> $O/sanitizer.txt 2>&1
done
grep -E "^=== |SUMMARY" $O/sanitizer.txt
timeout 900 python bench.py --timeline $O/overlap_timeline.json > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json, sys
d=json.loads(open(sys.argv[1]).read().splitlines()[-1]); o=d['overlap']
print("value", d['value'], "gather", d['roofline']['achieved'], "frac", d['roofline']['frac'], "e2e", d['e2e']['value'], "parity", d['parity']['exact'])
print(o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], "strict", o['hidden_frac_best'], "part", o['hidden_frac_partitioned']['value'], o['best']['shape'], o['best']['t_step_overlapped_ms'], o['consumer_roofline']['frac'])
PY
