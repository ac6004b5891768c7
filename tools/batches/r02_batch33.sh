#!/bin/bash
# ncu --set full of one gather launch with the final code (gathers at the maximum shared-memory carveout):
# refreshes roofline.traffic's source record (key config4_managed; the previous capture kept as *_previous)
O=gpurun_out/r02b33
mkdir -p $O
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o $O/prof_gather_managed python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > $O/prof_gather_managed.log 2>&1
cp profiles/r02/ncu_gather_summary.json $O/ncu_gather_summary.json
python tools/ncu_summary.py $O/prof_gather_managed.ncu-rep $O/ncu_gather_summary.json config4_managed \
    "ncu --set full, launch 4 of bench.py --steps 3 --warmup 3 (round 2 final code: managed host table, maximum shared-memory carveout)" > $O/ncu_summary_managed.log 2>&1
ncu -i $O/prof_gather_managed.ncu-rep --page raw --csv > $O/ncu_gather_managed_raw.csv 2>/dev/null
ncu -i $O/prof_gather_managed.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for k in ('launch__shared_mem_config_size','launch__occupancy_limit_shared_mem','sm__warps_active.avg.pct_of_peak_sustained_active'):
  for i,x in enumerate(h):
    if x==k: print(k, r[1][i], v[i])
"
rm -f $O/prof_gather_managed.ncu-rep
tail -25 $O/ncu_summary_managed.log
