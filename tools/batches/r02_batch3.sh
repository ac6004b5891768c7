#!/bin/bash
# round-2 GPU batch 3: ncu launch list, N > 1 readiness with ranks sharing one GPU (config 4 x 4 ranks,
# config 3 x 8 ranks, config 5 x 2 ranks, sharded cache x 2 ranks), sanitizers, bench config 4
O=gpurun_out/r02
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_config4.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_bench.log 2>&1 || \
ncu --metrics gpu__time_duration.sum --clock-control none --replay-mode application -c 400 --csv --log-file $O/launches_config4.csv \
    python bench.py --steps 4 --warmup 3 --no-baselines --no-overlap > $O/launches_bench_app.log 2>&1
run() {  # name nproc args...
  local name=$1 n=$2; shift 2
  DGZ_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 400)) bench.py --gpus $n "$@" > $O/$name.json 2> $O/$name.err
}
run bench_4ranks_same_gpu_config4 4 --steps 10 --warmup 3 --no-overlap
run bench_8ranks_same_gpu_config3 8 --config 3 --steps 10 --warmup 3 --no-overlap
run bench_2ranks_same_gpu_config5 2 --config 5 --row-bytes 512 --steps 6 --warmup 3 --oracle-budget 5
run bench_2ranks_same_gpu_cache20 2 --cache-frac 0.2 --steps 10 --warmup 3 --no-overlap
bash tools/sanitize.sh > $O/sanitizer.txt 2>&1
python bench.py --steps 20 --warmup 5 --timeline $O/overlap_timeline3.json > $O/bench_config4_b3.json 2> $O/bench_config4_b3.err
ls -la $O
