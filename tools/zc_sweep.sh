python -m pytest tests/test_gpu_zc_csr.py -x -q > gpurun_out/zc_tests.log 2>&1; tail -2 gpurun_out/zc_tests.log
for s in 0 16 32 64; do python bench.py --csr host --no-overlap --no-baselines --steps 20 --sampler-sms $s > gpurun_out/zc_s$s.json 2>>gpurun_out/zc_sweep.err; done
python - <<'PY'
import json
for s in (0,16,32,64):
    d=json.loads(open(f'gpurun_out/zc_s{s}.json').read().strip().splitlines()[-1])
    print(s, d['value'], d['roofline']['achieved'], d['latency_ms'], d['config']['pipeline'])
PY
