#!/bin/bash
# round-2 GPU batch 10: UVM baselines of the training example (test on config 1, numbers on config 4)
O=gpurun_out/r02
mkdir -p $O
python -m pytest tests/test_gpu_train_example.py -q -m gpu > $O/test_train_uvm.txt 2>&1
timeout 1500 python examples/graphsage_train.py --config 4 --steps 10 --modes zc,uvm,uvm_host > $O/train_uvm_config4.json 2> $O/train_uvm_config4.err
tail -3 $O/test_train_uvm.txt; tail -c 600 $O/train_uvm_config4.json
