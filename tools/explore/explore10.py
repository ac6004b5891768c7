"""Overlap with green-context SM partitions: fetch on k SMs, consumer on the rest."""
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
seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(16)]
rng = [gen.batch_rng_seed(c.seed, j) for j in range(16)]
A = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda"); B = torch.randn(8192, 8192, dtype=torch.bfloat16, device="cuda")
C = torch.empty(8192, 8192, dtype=torch.bfloat16, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)
N = 8
for fsms, fl in ((4, 2), (8, 2), (16, 2), (24, 2), (32, 2), (16, 1)):
    try:
        part = dgz.Partition(fsms, -1, fl)
    except Exception as e:
        out(fetch_sms=fsms, flags=fl, err=str(e)); continue
    f = MinibatchFetcher(tb, g, c.fanouts, c.batch, fetch_stream=part.fetch_stream)
    comp = part.compute_stream
    y = torch.empty((f.bufs[0].bounds[L - 1], c.dim), dtype=torch.float32, device="cuda")
    nb = sum(f.bufs[0].bounds[k] * c.fanouts[k] for k in range(L - 1)); cb = sum(f.bufs[0].bounds[k] for k in range(L - 1))
    def consumer(kind, mb, rep):
        with torch.cuda.stream(comp):
            if kind == "agg":
                dgz.aggregate_mean(mb.rows.view(torch.float32).view(-1), c.dim, mb.bufs.local[nb:], mb.bufs.cnt[cb:], c.fanouts[L - 1],
                                   mb.bufs.sizes_dev[L - 1:L], mb.bufs.bounds[L - 1], y, repeat=rep, stream=comp)
            else:
                for _ in range(rep): torch.matmul(A, B, out=C)
    def t_fetch():
        a, b = ev(), ev(); torch.cuda.synchronize(); a.record(f.stream)
        for i in range(N): f.fetch(seeds[i], rng[i])
        b.record(f.stream); torch.cuda.synchronize(); return a.elapsed_time(b) / N
    def t_cons(kind, mb, rep):
        a, b = ev(), ev(); torch.cuda.synchronize(); a.record(comp)
        for i in range(N): consumer(kind, mb, rep)
        b.record(comp); torch.cuda.synchronize(); return a.elapsed_time(b) / N
    def t_pipe(kind, rep):
        torch.cuda.synchronize(); mbs = [f.fetch(seeds[0], rng[0])]
        a, b = ev(), ev(); a.record(comp)
        for i in range(1, N + 1):
            nxt = f.fetch(seeds[i], rng[i]); cur = mbs[-1]
            comp.wait_event(cur.event); consumer(kind, cur, rep); f.release(cur, comp); mbs.append(nxt)
        comp.wait_event(mbs[-1].event); b.record(comp); torch.cuda.synchronize()
        return a.elapsed_time(b) / N
    for gs, gw in ((0, 0), (part.fetch_sms, 8), (part.fetch_sms * 2, 4), (part.fetch_sms * 4, 2)):
        f.cfg = dgz.gather_cfg(sm_count=gs, warps_per_cta=gw, flags=dgz.FLAG_DEEP) if gs else None
        out(fetch_sms=part.fetch_sms, grid=gs, warps=gw, t_fetch_alone=round(t_fetch(), 3))
    f.cfg = None
    tg = t_fetch()
    mb = f.fetch(seeds[0], rng[0]); mb.event.synchronize()
    ok = bool(torch.equal(mb.rows[:4].cpu(), torch.from_numpy(buf.numpy(0, c.table_bytes).reshape(c.n_nodes, R)[mb.bufs.ids[:4].cpu().numpy()])))
    for kind in ("agg", "gemm"):
        rep = 4
        for _ in range(3):
            tc = t_cons(kind, mb, rep); rep = max(1, round(rep * tg / tc))
        tc = t_cons(kind, mb, rep)
        to = t_pipe(kind, rep)
        out(fetch_sms=part.fetch_sms, compute_sms=part.compute_sms, consumer=kind, rep=rep, t_fetch=round(tg, 3), t_cons=round(tc, 3),
            t_step=round(to, 3), exposed=round(max(0, to - tc), 3), hidden=round(1 - max(0, to - tc) / tg, 3), rows_ok=ok)
    del f
    part.destroy()
