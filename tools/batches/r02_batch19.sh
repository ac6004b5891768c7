#!/bin/bash
# config-5 sweep, product path on the managed table vs the CPU-gather + cudaMemcpy baseline (16 and 2 threads)
O=gpurun_out/r02
mkdir -p $O
python tools/sweep_dma_vs_zc.py --managed > $O/sweep_dma_vs_zc_managed.jsonl 2> $O/sweep_managed.err
python tools/sweep_dma_vs_zc.py --managed --threads=2 --widths=64,128,256,512,1024,2048 > $O/sweep_dma_vs_zc_managed_2threads.jsonl 2> $O/sweep_managed2.err
cat $O/sweep_dma_vs_zc_managed.jsonl | head -60; tail -3 $O/sweep_managed.err
