#!/bin/bash
# ncu --set full of one gather launch of configs 2 and 3 (bench pipeline), for the per-config
# summaries in profiles/r01/ncu_gather_summary.json (one representative launch per config)
for c in 2 3; do
  ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
      -o gpurun_out/prof_gather_c$c python bench.py --config $c --steps 3 --warmup 3 --no-baselines --no-overlap \
      > gpurun_out/prof_gather_c$c.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
