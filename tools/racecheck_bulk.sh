#!/bin/bash
# compute-sanitizer racecheck over the BULK (TMA + mbarrier ring) gather: 512 B rows on 2 SMs
# (many ring wraps) and 40 KiB rows with the default 8 warps (more consumer warps than ring
# slots, the ADVICE r1 case), each checked against the source bytes.
cat > /tmp/san_bulk2.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
for R, rows, n, warps in ((512, 3000, 2000, 0), (40960, 64, 200, 0)):
    buf = dgz.HostBuffer(rows * R + 8192)
    gen.fill_table(buf.ptr, rows * R, R)
    t = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    ids = gen.random_ids(rows, n, 1)
    idx = torch.from_numpy(ids).cuda()
    out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
    dgz.gather(t, idx, out, cfg=dgz.gather_cfg(variant=4, sm_count=2, warps_per_cta=warps))
    torch.cuda.synchronize()
    src = buf.numpy(0, rows * R).reshape(rows, R)
    print("R", R, "exact", bool(np.array_equal(out.cpu().numpy().reshape(n, R), src[ids])), flush=True)
    t.unregister(); buf.free()
print("done")
PY
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 6 python /tmp/san_bulk2.py 2>&1 | tail -40
