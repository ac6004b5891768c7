# NEXT-4 training evaluation (examples/graphsage_train.py): fetch-partition sweep, then all modes
for s in 16 24 32 48; do python examples/graphsage_train.py --modes zc --fetch-sms $s --steps 20 >> gpurun_out/train_sweep.jsonl 2>>gpurun_out/train_sweep.err; done
python examples/graphsage_train.py --modes zc --fetch-sms 16 --sample-on fetch --steps 20 >> gpurun_out/train_sweep.jsonl 2>>gpurun_out/train_sweep.err
python examples/graphsage_train.py --steps 20 > gpurun_out/train_eval.json 2>>gpurun_out/train_sweep.err
python - <<'PY'
import json
for l in open('gpurun_out/train_sweep.jsonl'):
    d=json.loads(l); z=d['zc']; print(z['fetch_sms'], z['sampler_on'], z['step_ms'], z['fetch_alone_ms'], z['train_alone_ms'])
d=json.loads(open('gpurun_out/train_eval.json').read()); print({k:(v['step_ms'] if isinstance(v,dict) and 'step_ms' in v else v) for k,v in d.items()})
PY
