#!/bin/bash
# round-2 GPU batch 23 (the a7 layer on tcgen05): full GPU suite, the default bench with the layer as the
# overlap consumer, the consumer roofline, ncu --set full of one layer launch, launch list of the default
# bench command, sanitizers over the new kernel
O=gpurun_out/r02b23
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu > $O/gputest.txt 2>&1; tail -1 $O/gputest.txt
timeout 300 python tools/consumer_roofline.py > $O/consumer_roofline.jsonl 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:sage_mean --launch-skip 5 --launch-count 1 \
    -o $O/ncu_sage python tools/consumer_roofline.py --iters 2 > $O/ncu_sage.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_config4.csv \
    -k regex:'^(seeds|hop_sample|bitmap|local_all|gather|emit|scan|posmap)' \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_bench.log 2>&1
for tool in memcheck racecheck synccheck; do
  echo "=== $tool: gather variants + consumers" >> $O/sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/workers/san_variants.py >> $O/sanitizer.txt 2>&1
  tail -2 $O/sanitizer.txt
done
timeout 900 python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline.json > $O/bench_config4.json 2> $O/bench_config4.err
tail -c 600 $O/bench_config4.json
ls $O
