# training step with the fetch on contiguous vs spread partitions (examples/graphsage_train.py)
for s in 16 24; do
  python examples/graphsage_train.py --modes zc --fetch-sms $s --steps 20 --contiguous >> gpurun_out/train_spread.jsonl 2>>gpurun_out/train_spread.err
  python examples/graphsage_train.py --modes zc --fetch-sms $s --steps 20 >> gpurun_out/train_spread.jsonl 2>>gpurun_out/train_spread.err
done
python bench.py --no-baselines --steps 20 > gpurun_out/bench_ov3.json 2>gpurun_out/bench_ov3.err
python - <<'PY'
import json
for l in open('gpurun_out/train_spread.jsonl'):
    z=json.loads(l)['zc']; print(z['fetch_sms'], z['fetch_partition'], z['step_ms'], z['fetch_alone_ms'], z['train_alone_ms'])
d=json.loads(open('gpurun_out/bench_ov3.json').read().splitlines()[-1]); o=d['overlap']
print(d['value'], o['hidden_frac_best'])
for r in o['sweep']: print(r['partition'][:70], r['fetch_sms'], r['t_fetch_ms'], r['t_consumer_ms'], r['t_step_overlapped_ms'])
PY
