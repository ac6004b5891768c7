"""Row-width sweep of the PRODUCT path (dgz_order_ids + dgz_gather_perm, default launch): useful
GB/s for 256 MiB of uniformly random distinct rows per width and table base offset, over the
56.9 GB buffer.  Complements sweep_rowwidth.py (which compares the kernel variants)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
total = gen.CONFIGS[4].table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total + 4096, 9)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
for R in gen.SWEEP_ROW_BYTES:
    for base in (0, 4):
        rows = (total - base) // R
        n = min(rows, (256 << 20) // R)
        tb = dgz.register_table(buf.ptr + base, rows, R // 4 if R % 4 == 0 else R, dgz.F32 if R % 4 == 0 else dgz.U8)
        ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 7 + base)).cuda()
        srt, pos = dgz.order_ids(ids, rows)
        for _ in range(2): dgz.gather_perm(tb, srt, pos, outd, n=n)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(3): dgz.gather_perm(tb, srt, pos, outd, n=n)
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b) / 3
        print(json.dumps({"R": R, "base": base, "n": n, "gbs": round(n * R / t / 1e6, 2), "mrows_s": round(n / t / 1e3, 1)}), flush=True)
        tb.unregister()
