#!/bin/bash
# round-2 GPU batch 14: the managed host table (DGZ_HOST_MANAGED) -- parity, bench, small-row study, ncu
O=gpurun_out/r02
mkdir -p $O
python -m pytest tests/test_gpu_managed.py tests/test_gpu_parity.py -q -m gpu > $O/test_managed.txt 2>&1
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline14.json > $O/bench_config4_managed.json 2> $O/bench_config4_managed.err
python bench.py --steps 20 --warmup 5 --host-table registered --no-overlap > $O/bench_config4_registered.json 2> $O/bench_config4_registered.err
python tools/smallrow_study.py A B --managed > $O/smallrow_study_managed.jsonl 2> $O/smallrow_study_managed.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcnode_gpc.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_gcc.sum,pcie__read_bytes.sum,syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:gather_segment_kernel --csv --log-file $O/smallrow_ncu_managed.csv python tools/smallrow_study.py B --ncu --managed > $O/smallrow_ncu_managed.log 2>&1
for spec in "128 f32 0" "64 f32 0" "256 f32 0"; do
  set -- $spec
  python bench.py --config 5 --row-bytes $1 --dtype $2 --base $3 --steps 10 --warmup 3 --oracle-budget 10 \
      > $O/bench_config5_managed_R$1.json 2> $O/bench_config5_managed_R$1.err
done
tail -3 $O/test_managed.txt
