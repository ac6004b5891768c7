#!/bin/bash
# round-2 GPU batch 9: overlap leg with whole-GPU consumer candidates (more fetch SMs, 1 warp each)
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline9.json > $O/bench_config4_b9.json 2> $O/bench_config4_b9.err
tail -c 300 $O/bench_config4_b9.json
