#!/bin/bash
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --cache-frac 0.2 --no-overlap > $O/bench_config4_cache20_managed.json 2> $O/bench_cache20_managed.err
python -m pytest tests -m gpu -q -k "cache or managed or bench" > $O/test_b21.txt 2>&1
tail -c 600 $O/bench_config4_cache20_managed.json; tail -2 $O/test_b21.txt
