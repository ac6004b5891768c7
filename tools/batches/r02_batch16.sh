#!/bin/bash
# managed table: launch-shape sweep; overlap leg with the sampler in the whole-GPU consumer's stream;
# 2 ranks x 20 GB managed tables on one GPU (is the two-process failure size-related?)
O=gpurun_out/r02
mkdir -p $O
python tools/managed_shape_sweep.py > $O/managed_shape_sweep.jsonl 2> $O/managed_shape_sweep.err
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline16.json > $O/bench_config4_b16.json 2> $O/bench_config4_b16.err
DGZ_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29612 bench.py --gpus 2 --config 5 --row-bytes 512 --table-gb 20 --host-table managed --steps 5 --warmup 3 \
    --oracle-budget 2 > $O/bench_2ranks_managed_20gb.json 2> $O/bench_2ranks_managed_20gb.err
cat $O/managed_shape_sweep.jsonl; tail -c 300 $O/bench_2ranks_managed_20gb.json; grep -m2 -E "Error" $O/bench_2ranks_managed_20gb.err
