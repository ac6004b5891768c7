"""compute-sanitizer target (test infrastructure: checks against the oracle): every gather variant
(SEGMENT, NAIVE, SHIFT, BULK) and the sorted gather at three row widths (tools/sanitize.sh)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
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
