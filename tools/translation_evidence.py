"""Same number of sorted 512 B rows gathered from a 1 GB and from a 56.9 GB footprint: profile both
launches with ncu to show the GPU page-walk traffic (DRAM / L2 reads not issued by the SMs) grow
with the footprint while the payload stays identical."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
total = gen.CONFIGS[4].table_bytes; R = 512; n = 800_000
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 3)
tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
for gb in (1.0, 56.8):
    rows = int(gb * 1e9) // R
    ids = torch.sort(torch.from_numpy(gen.distinct_ids(rows, n, 77)).cuda()).values
    pos = torch.arange(n, dtype=torch.int64, device="cuda")
    for _ in range(2):
        dgz.gather_perm(tb, ids, pos, outd, n=n)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dgz.gather_perm(tb, ids, pos, outd, n=n); b.record(); torch.cuda.synchronize()
    print(f"footprint {gb} GB: {n * R / a.elapsed_time(b) / 1e6:.2f} GB/s", flush=True)
