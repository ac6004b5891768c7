cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_sage.py -q -x 2>&1 | tail -1
timeout 120 python tools/consumer_roofline.py | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['kernel'], d['ms'], d['hbm_gbs'])"
timeout 900 python bench.py --no-baselines > gpurun_out/bench_ov4.json 2> gpurun_out/bench_ov4.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_ov4.json').read().splitlines()[-1]); o=d['overlap']
print(d['value'], o['t_fetch_ms'], o['consumer_repeat'], o['t_consumer_ms'], o['hidden_frac_best'], o['hidden_frac_partitioned'], o['consumer_roofline'])
for r in o['sweep']:
    print(r.get('shape'), r.get('t_fetch_ms'), r.get('t_consumer_ms'), r.get('t_step_overlapped_ms'), r.get('exposed_fetch_ms'))
PY
