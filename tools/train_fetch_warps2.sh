# training step with larger fetch partitions and few warps per SM
for sw in "40 2" "48 1" "48 2" "64 1" "32 2"; do
  set -- $sw
  python examples/graphsage_train.py --modes zc --steps 20 --fetch-sms $1 --fetch-warps $2 >> gpurun_out/train_eval_fetch_warps2.jsonl 2>/dev/null
done
python - <<'PY'
import json
for l in open("gpurun_out/train_eval_fetch_warps2.jsonl"):
    z = json.loads(l)["zc"]; print(z["fetch_sms"], z["fetch_warps_per_sm"], z["step_ms"], z["fetch_alone_ms"], z["train_alone_ms"])
PY
