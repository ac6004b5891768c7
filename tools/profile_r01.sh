#!/bin/bash
# ncu evidence for round 1 (run on the GPU box via gpurun). Never a multi-rank command.
set -x
mkdir -p gpurun_out
ncu --query-metrics > gpurun_out/ncu_query_metrics.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 2 \
    -o gpurun_out/prof_gather python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > gpurun_out/prof_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hop_sample_kernel -s 6 -c 3 \
    -o gpurun_out/prof_sampler python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > gpurun_out/prof_sampler.log 2>&1
ls -la gpurun_out
