#!/bin/bash
O=gpurun_out/r02
mkdir -p $O
python tools/cache_managed_shapes.py > $O/cache_managed_shapes.jsonl 2> $O/cache_managed_shapes.err
cat $O/cache_managed_shapes.jsonl; tail -3 $O/cache_managed_shapes.err
