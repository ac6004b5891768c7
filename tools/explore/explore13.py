"""What slows a co-running gather: SM issue contention or the memory system?
Full-GPU sorted gather (default) alone, then beside (a) a pure-ALU spin load filling every SM,
(b) the HBM-bound aggregation consumer, (c) a cuBLAS GEMM."""
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
gs = torch.cuda.Stream(priority=-1); cs = torch.cuda.Stream()
sink = torch.zeros(1, device="cuda")
A = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda"); B = torch.randn_like(A); C = torch.empty_like(A)
X = torch.randn(800_000, 128, device="cuda"); Y = torch.empty(200_000, 128, device="cuda")
idxr = torch.randint(0, 800_000, (200_000, 5), device="cuda")
CFG = [None]
def gather():
    with torch.cuda.stream(gs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(gs); dgz.gather_perm(tb, ids, pos, outd, n=n, stream=gs, cfg=CFG[0]); b.record(gs)
    return a, b
def load(kind):
    with torch.cuda.stream(cs):
        if kind == "spin":
            dgz.probe_spin(148 * 6, 256, 400_000, sink, stream=cs)
        elif kind == "hbm":
            for _ in range(60): Y.copy_(X[idxr].mean(1))
        elif kind == "gemm":
            for _ in range(20): torch.matmul(A, B, out=C)
cfgs = {"default": None,
        "148x8_deep": dgz.gather_cfg(sm_count=148, warps_per_cta=8, flags=dgz.FLAG_DEEP),
        "148x16": dgz.gather_cfg(sm_count=148, warps_per_cta=16),
        "296x4_deep": dgz.gather_cfg(sm_count=148, warps_per_cta=4, ctas_per_sm=2, flags=dgz.FLAG_DEEP),
        "bulk_148x8": dgz.gather_cfg(variant=dgz.GATHER_BULK, sm_count=148, warps_per_cta=8),
        "bulk_148x4": dgz.gather_cfg(variant=dgz.GATHER_BULK, sm_count=148, warps_per_cta=4)}
for name, cfg in cfgs.items():
    CFG[0] = cfg
    for kind in ("none", "spin", "gemm"):
        for rep in range(2):
            torch.cuda.synchronize()
            if kind != "none": load(kind)
            a, b = gather()
            torch.cuda.synchronize()
        t = a.elapsed_time(b)
        out(cfg=name, load=kind, gather_ms=round(t, 3), gbs=round(n * R / t / 1e6, 2))
