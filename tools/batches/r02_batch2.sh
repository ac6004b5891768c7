#!/bin/bash
# round-2 GPU batch 2: bench config 4 (steady-state overlap, e2e diagnostics), the ncu launch list and
# one --set full capture of the gather, 8 ranks sharing one GPU (N > 1 readiness), the sharded cache
# mode, config-5 points through bench.py, and the reference arm.
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline2.json > $O/bench_config4_b2.json 2> $O/bench_config4_b2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o $O/prof_gather python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > $O/prof_gather.log 2>&1
python tools/ncu_summary.py $O/prof_gather.ncu-rep $O/ncu_gather_summary.json config4 \
    "ncu --set full, launch 4 of bench.py --steps 3 --warmup 3 (round 2)" > $O/ncu_summary.log 2>&1
ncu -i $O/prof_gather.ncu-rep --page raw --csv > $O/ncu_gather_full_raw.csv 2>/dev/null
rm -f $O/prof_gather.ncu-rep
DGZ_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --gpus 8 --steps 10 --warmup 3 --no-overlap > $O/bench_8ranks_same_gpu.json 2> $O/bench_8ranks_same_gpu.err
python bench.py --steps 20 --warmup 5 --cache-frac 0.2 --no-overlap > $O/bench_config4_cache20.json 2> $O/bench_config4_cache20.err
for spec in "128 f32 0" "66 f16 4" "1030 f16 0" "400 f32 0"; do
  set -- $spec
  python bench.py --config 5 --row-bytes $1 --dtype $2 --base $3 --steps 10 --warmup 3 --oracle-budget 10 \
      > $O/bench_config5_R$1_$2_b$3.json 2> $O/bench_config5_R$1_$2_b$3.err
done
python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
ls -la $O
