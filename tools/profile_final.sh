#!/bin/bash
# Final round-1 ncu evidence for the default bench pipeline (run on the GPU box via gpurun).
# The launch list uses --sampler-sms 0 (ncu cannot prepare every kernel of a green-context
# stream for the metric pass); the kernels and their shares are the same.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 6 --warmup 3 --no-baselines --no-overlap --sampler-sms 0 > gpurun_out/launches_final_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o gpurun_out/prof_gather_final python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > gpurun_out/prof_gather_final.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:hop_sample_kernel -s 6 -c 3 \
    -o gpurun_out/prof_sampler_final python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap --sampler-sms 0 > gpurun_out/prof_sampler_final.log 2>&1
