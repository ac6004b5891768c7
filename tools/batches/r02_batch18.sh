#!/bin/bash
# managed-table launch rule (4 warps per SM for rows of >= 2 lines): bench config 4 and a config-5 point
O=gpurun_out/r02
mkdir -p $O
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline18.json > $O/bench_config4_b18.json 2> $O/bench_config4_b18.err
python bench.py --config 5 --row-bytes 256 --steps 10 --warmup 3 --oracle-budget 5 > $O/bench_config5_managed_R256_b18.json 2> $O/b18c5.err
python -m pytest tests/test_gpu_managed.py tests/test_gpu_consumer_merge.py -q -m gpu > $O/test_b18.txt 2>&1
tail -c 300 $O/bench_config4_b18.json; tail -2 $O/test_b18.txt
