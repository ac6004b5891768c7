#!/bin/bash
# round-2 GPU batch 6: overlap leg with the whole-GPU consumer placement
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline6.json > $O/bench_config4_b6.json 2> $O/bench_config4_b6.err
tail -c 300 $O/bench_config4_b6.json
