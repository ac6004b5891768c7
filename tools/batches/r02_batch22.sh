#!/bin/bash
# ncu evidence for the managed default: --set full of one gather launch, the launch list (libdgz kernels)
O=gpurun_out/r02
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o $O/prof_gather_managed python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > $O/prof_gather_managed.log 2>&1
cp profiles/r02/ncu_gather_summary.json $O/ncu_gather_summary.json
python tools/ncu_summary.py $O/prof_gather_managed.ncu-rep $O/ncu_gather_summary.json config4_managed \
    "ncu --set full, launch 4 of bench.py --steps 3 --warmup 3 (round 2, managed host table)" > $O/ncu_summary_managed.log 2>&1
ncu -i $O/prof_gather_managed.ncu-rep --page raw --csv > $O/ncu_gather_managed_raw.csv 2>/dev/null
rm -f $O/prof_gather_managed.ncu-rep
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4_managed.csv \
    -k regex:'^(seeds|hop_sample|bitmap|local_all|gather|emit|scan|posmap)' \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_managed.log 2>&1
cat $O/ncu_summary_managed.log | tail -25
