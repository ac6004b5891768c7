#!/bin/bash
# UVM-mapped host memory vs cudaHostRegister for the translation-bound gathers
O=gpurun_out/r02
mkdir -p $O
timeout 1500 python tools/uvm_host_study.py reg managed hmm > $O/uvm_host_study.jsonl 2> $O/uvm_host_study.err
cat $O/uvm_host_study.jsonl; tail -5 $O/uvm_host_study.err
