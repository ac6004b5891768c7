#!/bin/bash
# What the driver runs at round end, in one gpurun call:
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/round_end_check.sh'
set -o pipefail
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/rc_pytest_gpu.log 2>&1; echo "pytest -m gpu rc=$?"; tail -1 gpurun_out/rc_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/rc_bench_ref.json 2> gpurun_out/rc_bench_ref.err; echo "reference rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/rc_bench.json").read().splitlines()[-1])
r = json.loads(open("gpurun_out/rc_bench_ref.json").read().splitlines()[-1])
print("ours:", d["value"], d["unit"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["value"], "launches", d["gpu_launches"],
      "parity", d["parity"]["exact"], "clocks", d["clocks"]["reasons"])
print("reference:", r["value"], r["unit"], "ratio", round(d["value"] / r["value"], 1))
PY
