"""Overlap: what slows the gather when a consumer runs beside it?  (SM slots vs memory system)"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
from paper_2103_03330_b200.pipeline import MinibatchFetcher

def out(**kw): print(json.dumps(kw), flush=True)
torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes; L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
f = MinibatchFetcher(tb, g, c.fanouts, c.batch)
seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(16)]
rng = [gen.batch_rng_seed(c.seed, j) for j in range(16)]
comp = torch.cuda.Stream()
y = torch.empty((f.bufs[0].bounds[L - 1], c.dim), dtype=torch.float32, device="cuda")
nb = sum(f.bufs[0].bounds[k] * c.fanouts[k] for k in range(L - 1)); cb = sum(f.bufs[0].bounds[k] for k in range(L - 1))
A = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda"); B = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
C = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
N = 8

def consumer(kind, mb, rep):
    with torch.cuda.stream(comp):
        if kind.startswith("agg"):
            cps = int(kind[3:])
            dgz.aggregate_mean(mb.rows.view(torch.float32).view(-1), c.dim, mb.bufs.local[nb:], mb.bufs.cnt[cb:], c.fanouts[L - 1],
                               mb.bufs.sizes_dev[L - 1:L], mb.bufs.bounds[L - 1], y, repeat=rep, ctas_per_sm=cps, stream=comp)
        else:
            for _ in range(rep):
                torch.matmul(A, B, out=C)

def t_alone_fetch():
    a, b = ev(), ev(); torch.cuda.synchronize(); a.record(f.stream)
    for i in range(N): f.fetch(seeds[i], rng[i])
    b.record(f.stream); torch.cuda.synchronize(); return a.elapsed_time(b) / N

def t_alone_cons(kind, mb, rep):
    a, b = ev(), ev(); torch.cuda.synchronize(); a.record(comp)
    for i in range(N): consumer(kind, mb, rep)
    b.record(comp); torch.cuda.synchronize(); return a.elapsed_time(b) / N

def t_pipe(kind, rep):
    torch.cuda.synchronize()
    mbs = [f.fetch(seeds[0], rng[0])]
    a, b = ev(), ev(); a.record(comp)
    gev = []
    for i in range(1, N + 1):
        nxt = f.fetch(seeds[i], rng[i]); cur = mbs[-1]
        comp.wait_event(cur.event); consumer(kind, cur, rep); f.release(cur, comp); mbs.append(nxt)
    comp.wait_event(mbs[-1].event); b.record(comp); torch.cuda.synchronize()
    return a.elapsed_time(b) / N

for gcfg_name, gcfg in (("default", None), ("48x2deep", dgz.gather_cfg(sm_count=48, warps_per_cta=2, flags=dgz.FLAG_DEEP)),
                        ("16x4deep", dgz.gather_cfg(sm_count=16, warps_per_cta=4, flags=dgz.FLAG_DEEP))):
    f.cfg = gcfg
    tg = t_alone_fetch()
    mb = f.fetch(seeds[0], rng[0]); mb.event.synchronize()
    for kind in ("agg0", "agg2", "gemm"):
        rep = 4
        for _ in range(3):
            tc = t_alone_cons(kind, mb, rep); rep = max(1, round(rep * tg / tc))
        tc = t_alone_cons(kind, mb, rep)
        to = t_pipe(kind, rep)
        out(gather=gcfg_name, consumer=kind, rep=rep, t_fetch=round(tg, 3), t_cons=round(tc, 3), t_step=round(to, 3),
            exposed=round(to - tc, 3), hidden=round(1 - max(0, to - tc) / tg, 3))
