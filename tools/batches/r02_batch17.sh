#!/bin/bash
O=gpurun_out/r02
mkdir -p $O
python tools/managed_shape_sweep.py > $O/managed_shape_sweep.jsonl 2> $O/managed_shape_sweep.err
cat $O/managed_shape_sweep.jsonl; tail -3 $O/managed_shape_sweep.err
