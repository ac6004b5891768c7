#!/bin/bash
# NEXT-4 fig:eval_overall analogue with the UVM baselines: all five strategies on config 4, 20 steps
O=gpurun_out/r02
mkdir -p $O
timeout 2000 python examples/graphsage_train.py --config 4 --steps 20 --modes zc,dma,hbm,uvm,uvm_host > $O/train_eval_uvm_config4.json 2> $O/train_eval_uvm_config4.err
tail -c 1500 $O/train_eval_uvm_config4.json
