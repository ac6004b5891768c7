#!/bin/bash
# Re-profile the default (sorted, 148 CTAs x 2 warps, 16 lines in flight per lane) gather; 2-rank bench on one GPU.
set -x
ncu --set full --clock-control none --import-source on -k regex:gather_segment_kernel -s 3 -c 1 \
    -o gpurun_out/prof_gather_deep python bench.py --steps 3 --warmup 3 --no-baselines --no-overlap > gpurun_out/prof_gather_deep.log 2>&1
DGZ_BENCH_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-overlap > gpurun_out/bench_2ranks_samegpu.json 2> gpurun_out/bench_2ranks_samegpu.err
