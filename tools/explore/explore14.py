"""Gather and an ALU spin load on DISJOINT green-context partitions: is the interference shared
hardware (clocks / GPC / MMU) or SM issue?"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
def out(**kw): print(json.dumps(kw), flush=True)
torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
n = 800_000
ids = torch.sort(torch.from_numpy(gen.distinct_ids(c.n_nodes, n, 5)).cuda()).values
pos = torch.arange(n, dtype=torch.int64, device="cuda")
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
sink = torch.zeros(1, device="cuda")
for k in (32, 74, 116):
    part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD)
    gs, cs = part.fetch_stream, part.compute_stream
    for kind in ("none", "spin", "spin_small"):
        for rep in range(2):
            torch.cuda.synchronize()
            if kind == "spin":
                dgz.probe_spin(part.compute_sms * 6, 256, 600_000, sink, stream=cs)
            if kind == "spin_small":
                dgz.probe_spin(part.compute_sms, 64, 2_000_000, sink, stream=cs)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(gs); dgz.gather_perm(tb, ids, pos, outd, n=n, stream=gs); b.record(gs)
            torch.cuda.synchronize()
        t = a.elapsed_time(b)
        out(gather_sms=part.fetch_sms, spin_sms=part.compute_sms, load=kind, gather_ms=round(t, 3), gbs=round(n * R / t / 1e6, 2))
    part.destroy()
