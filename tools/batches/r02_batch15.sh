#!/bin/bash
# round-2 GPU batch 15: unsorted lists on the managed table, training with the managed table, the full
# GPU suite, 2 ranks with per-rank managed tables
O=gpurun_out/r02
mkdir -p $O
python tools/smallrow_study.py B --managed --unsorted > $O/smallrow_study_managed_unsorted.jsonl 2> $O/smallrow_unsorted.err
timeout 1500 python examples/graphsage_train.py --config 4 --steps 20 --modes zc,dma --host-table managed > $O/train_managed_config4.json 2> $O/train_managed.err
python -m pytest tests -m gpu -q > $O/gputest_b15.txt 2>&1
DGZ_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-overlap > $O/bench_2ranks_managed.json 2> $O/bench_2ranks_managed.err
cat $O/smallrow_study_managed_unsorted.jsonl; tail -c 800 $O/train_managed_config4.json; tail -2 $O/gputest_b15.txt
