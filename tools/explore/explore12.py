"""Plain dgz_gather on random (unsorted) rows of the 56.9 GB table: auto address-ordering."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
for n in (100_000, 800_000):
    ids = torch.from_numpy(gen.distinct_ids(c.n_nodes, n, 9)).cuda()
    out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
    for name, fn in (("dgz_gather (auto order)", lambda: dgz.gather(tb, ids, out)),
                     ("dgz_gather_ex unordered", lambda: dgz.gather(tb, ids, out, cfg=dgz.gather_cfg()))):
        for _ in range(2): fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(4): fn()
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 4
        print(json.dumps({"n": n, "path": name, "ms": round(t, 3), "gbs": round(n * R / t / 1e6, 2)}), flush=True)
