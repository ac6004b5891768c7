#!/bin/bash
# round-2 GPU batch 1: new bench modes, multi-rank bench / training tests, small-row study, store widths
mkdir -p gpurun_out/r02
python -m pytest tests/test_gpu_bench_ranks.py tests/test_gpu_train_example.py -q -m gpu > gpurun_out/r02/tests_bench_train.txt 2>&1
python bench.py --steps 20 --warmup 5 --timeline gpurun_out/r02/overlap_timeline.json > gpurun_out/r02/bench_config4.json 2> gpurun_out/r02/bench_config4.err
python tools/smallrow_study.py A B > gpurun_out/r02/smallrow_study.jsonl 2> gpurun_out/r02/smallrow_study.err
python tools/sweep_store_width.py > gpurun_out/r02/sweep_store_width.jsonl 2> gpurun_out/r02/sweep_store_width.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_sectors_srcnode_gpc.sum,lts__t_sectors_srcunit_tex.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_gcc.sum,pcie__read_bytes.sum,syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum
timeout 1200 ncu --metrics $M --clock-control none -k regex:gather_segment_kernel --csv --log-file gpurun_out/r02/smallrow_ncu.csv python tools/smallrow_study.py A B --ncu > gpurun_out/r02/smallrow_ncu.log 2>&1
tail -2 gpurun_out/r02/tests_bench_train.txt
