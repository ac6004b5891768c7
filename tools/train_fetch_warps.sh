# training step vs the fetch partition's SMs x warps (spread SMs, work-counter batches; examples/graphsage_train.py)
for sw in "16 2" "16 3" "24 2" "32 2" "32 3" "16 8" "24 8"; do
  set -- $sw
  python examples/graphsage_train.py --modes zc --steps 20 --fetch-sms $1 --fetch-warps $2 >> gpurun_out/train_eval_fetch_warps.jsonl 2>/dev/null
done
python - <<'PY'
import json
for l in open("gpurun_out/train_eval_fetch_warps.jsonl"):
    z = json.loads(l)["zc"]; print(z["fetch_sms"], z["fetch_warps_per_sm"], z["step_ms"], z["fetch_alone_ms"], z["train_alone_ms"])
PY
