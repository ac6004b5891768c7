#!/bin/bash
# compute-sanitizer on config 1: memcheck / racecheck / synccheck over the smoke
# path (sampler + SEGMENT gather) and the BULK (smem ring + mbarrier) and NAIVE/SHIFT gathers.
cat > /tmp/san_bulk.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import dgz_inputs as gen, oracle
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
for R, base in ((512, 0), (2408, 8), (100, 4)):
    rows = 3000
    buf = dgz.HostBuffer(rows * R + 8192)
    gen.fill_table(buf.ptr + base, rows * R, R)
    t = dgz.register_table(buf.ptr + base, rows, R // 4, dgz.F32)
    idx = gen.random_ids(rows, 2000, 1)
    want, _ = oracle.gather(buf.numpy(base, rows * R), R, idx)
    out = torch.empty(2000 * R, dtype=torch.uint8, device="cuda")
    ids = torch.from_numpy(idx).cuda()
    for v in (1, 2, 3, 4):
        dgz.gather(t, ids, out, cfg=dgz.gather_cfg(variant=v, sm_count=4))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), (R, v)
    o = np.argsort(idx, kind="stable")
    dgz.gather_perm(t, torch.from_numpy(idx[o]).cuda(), torch.from_numpy(o.astype(np.int64)).cuda(), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    t.unregister(); buf.free()
print("bulk/segment/naive/shift ok")
PY
for tool in memcheck racecheck synccheck initcheck; do
  echo "=== $tool: smoke (sampler + segment gather, config 1)"
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python __graft_entry__.py --smoke 2>&1 | tail -4
  echo "=== $tool: gather variants"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_bulk.py 2>&1 | tail -4
done
