#!/bin/bash
# round-2 GPU batch 4: ncu launch lists (the default pipelined bench fails to profile its first sampler
# kernel on the 8-SM green-context partition; the sequential pipeline is profiled instead), the full GPU
# test suite, smoke
O=gpurun_out/r02
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4_seq.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap --sampler-sms 0 > $O/launches_seq.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seeds_small -c 3 --csv --log-file $O/launches_seeds_small_only.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_seeds_only.log 2>&1
python -m pytest tests -m gpu -q > $O/gputest.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.txt 2>&1
tail -3 $O/gputest.txt
