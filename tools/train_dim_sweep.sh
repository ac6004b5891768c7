# fig:eval_sweep analogue: GraphSAGE training on the products-shaped graph with the
# feature dimension swept, fed by zero-copy vs the CPU-gather + cudaMemcpy baseline (one GPU)
for d in 100 512 2048; do
  python examples/graphsage_train.py --config 3 --dim $d --modes zc,dma --steps 10 >> gpurun_out/train_dim_sweep.jsonl 2>>gpurun_out/train_dim_sweep.err
done
python - <<'PY'
import json
for l in open('gpurun_out/train_dim_sweep.jsonl'):
    d = json.loads(l)
    print(d["dim"], d["zc"]["step_ms"], d["zc"]["fetch_alone_ms"], d["zc"]["train_alone_ms"], d["dma"]["step_ms"], d["speedup_zc_over_dma"])
PY
