#!/bin/bash
# Round-1 (session 2, final kernel) ncu evidence for the default bench pipeline, after the launch-shape rule and
# the cache-hint argument changed the gather kernel.  Same recipe as profile_final.sh.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_s3.csv \
    python bench.py --steps 6 --warmup 3 --no-baselines --no-overlap --sampler-sms 0 > gpurun_out/launches_s3_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o gpurun_out/prof_gather_s3 python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > gpurun_out/prof_gather_s3.log 2>&1
ls -la gpurun_out/
