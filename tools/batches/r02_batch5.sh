#!/bin/bash
# round-2 GPU batch 5: bench config 4 with the RTT and All-in-GPU context legs (twice), the default
# command's launch list restricted to libdgz kernels
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline5.json > $O/bench_config4_b5.json 2> $O/bench_config4_b5.err
python bench.py --steps 20 --warmup 5 --no-overlap > $O/bench_config4_b5b.json 2> $O/bench_config4_b5b.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4_dgz.csv \
    -k regex:'^(seeds|hop_sample|bitmap|local_all|gather|emit|scan|posmap)' \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_dgz.log 2>&1
tail -c 400 $O/bench_config4_b5.json
