#!/bin/bash
# after the carveout change: full GPU suite, sanitizers, the layer's roofline + ncu, configs 2 / 3 / 5 bench lines
O=gpurun_out/r02b28; mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu > $O/gputest.txt 2>&1; tail -1 $O/gputest.txt
timeout 300 python tools/consumer_roofline.py > $O/consumer_roofline.jsonl 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sage_mean --launch-skip 5 --launch-count 1 \
    -o $O/ncu_sage python tools/consumer_roofline.py --iters 2 > $O/ncu_sage.log 2>&1
for tool in memcheck synccheck; do
  echo "=== $tool" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_variants.py >> $O/sanitizer.txt 2>&1
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py --smoke >> $O/sanitizer.txt 2>&1
done
grep -E "ERROR SUMMARY|ok" $O/sanitizer.txt
for c in 2 3; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > $O/bench_config$c.json 2> $O/bench_config$c.err
  tail -c 400 $O/bench_config$c.json; echo
done
timeout 900 python bench.py --config 5 --row-bytes 128 --steps 10 --warmup 3 --oracle-budget 5 > $O/bench_config5_R128.json 2> $O/bench_config5_R128.err
tail -c 300 $O/bench_config5_R128.json
