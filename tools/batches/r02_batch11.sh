#!/bin/bash
# diagnose: zero-copy training overlap (r01: 9.7 ms per step; batch 10: 14.4)
O=gpurun_out/r02
mkdir -p $O
timeout 900 python examples/graphsage_train.py --config 4 --steps 20 --modes zc > $O/train_zc_dyn.json 2> $O/train_zc_dyn.err
DGZ_TRAIN_STATIC=1 timeout 900 python examples/graphsage_train.py --config 4 --steps 20 --modes zc > $O/train_zc_static.json 2> $O/train_zc_static.err
timeout 900 python examples/graphsage_train.py --config 4 --steps 20 --modes zc --sample-on fetch > $O/train_zc_dyn_samplefetch.json 2> $O/train_zc_dyn_samplefetch.err
for f in $O/train_zc_*.json; do echo $f; tail -c 400 $f; echo; done
