"""NEXT-1: HBM hot-row cache on a power-law (skewed) papers100M-shaped graph, one B200.

Rows are ranked by in-degree (how often a sampler can reach them); the top fraction is cached in
HBM; each minibatch is sampled on the GPU and fetched with dgz_gather_cached (address order).
Reports effective GB/s (useful bytes / fetch time), the hit rate (rows served from HBM) and the
PCIe bytes avoided, next to the uncached fetch and the All-in-HBM reference.
"""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz

def out(**kw): print(json.dumps(kw), flush=True)
def ev(): return torch.cuda.Event(enable_timing=True)
torch.cuda.set_device(0)
alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
c = gen.CONFIGS[4]; R = c.row_bytes; L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
t0 = time.time()
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed, skew_alpha=alpha)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
indeg = torch.bincount(g.cols.long(), minlength=c.n_nodes)
order = torch.argsort(indeg, descending=True)
out(step="graph", alpha=alpha, s=round(time.time() - t0, 1), edges=int(off[-1]),
    top1pct_edge_share=round(float(indeg[order[:c.n_nodes // 100]].sum()) / int(off[-1]), 3))
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
mbs = []
for j in range(8):
    seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda()
    dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, j), bufs)
    torch.cuda.synchronize()
    n = int(bufs.sizes_host[-1])
    mbs.append((bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone(), n))
nmean = sum(m[2] for m in mbs) / len(mbs)
outd = torch.empty(max(m[2] for m in mbs) * R, dtype=torch.uint8, device="cuda")

def timeit(fn):
    for m in mbs[:2]: fn(*m)
    a, b = ev(), ev(); torch.cuda.synchronize(); a.record()
    for m in mbs: fn(*m)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / len(mbs)

t = timeit(lambda ids, pos, n: dgz.gather_perm(tb, ids, pos, outd, n=n))
out(step="uncached", rows_per_batch=round(nmean), ms=round(t, 3), gbs=round(nmean * R / t / 1e6, 2))
for frac in (0.01, 0.05, 0.10, 0.20):
    k = int(c.n_nodes * frac)
    cache = dgz.HotRowCache(tb, order[:k].contiguous())
    torch.cuda.synchronize()
    hits = [float((cache.slot_map[m[0]] >= 0).float().mean()) for m in mbs]
    t = timeit(lambda ids, pos, n: cache.gather(ids, outd, dst_pos=pos, n=n))
    out(step="cached", frac=frac, cache_gb=round(k * R / 1e9, 2), hit_rate=round(float(np.mean(hits)), 4), ms=round(t, 3),
        gbs=round(nmean * R / t / 1e6, 2), pcie_gb_per_batch=round(nmean * R * (1 - np.mean(hits)) / 1e9, 4))
    del cache; torch.cuda.empty_cache()
# All-in-HBM reference: the whole 56.9 GB table in HBM
dev_table = torch.empty(c.table_bytes, dtype=torch.uint8, device="cuda")
dev_table.copy_(torch.from_numpy(buf.numpy(0, c.table_bytes)))
dt = dgz.DeviceTable(dev_table.data_ptr(), c.n_nodes, c.dim, dgz.F32)
t = timeit(lambda ids, pos, n: dgz.gather_perm(dt, ids, pos, outd, n=n))
out(step="all_in_hbm", ms=round(t, 3), gbs=round(nmean * R / t / 1e6, 2), note="default HBM-table launch (148 x 4 CTAs x 16 warps)")
for cps, w in ((2, 16), (4, 8), (8, 8)):
    t = timeit(lambda ids, pos, n: dgz.gather_perm(dt, ids, pos, outd, n=n, cfg=dgz.gather_cfg(warps_per_cta=w, ctas_per_sm=cps)))
    out(step="all_in_hbm", ctas_per_sm=cps, warps=w, ms=round(t, 3), gbs=round(nmean * R / t / 1e6, 2))
m = mbs[0]
dgz.gather_perm(dt, m[0], m[1], outd, n=m[2]); ref = outd[:m[2] * R].clone()
dgz.gather_perm(tb, m[0], m[1], outd, n=m[2]); torch.cuda.synchronize()
out(step="check", equal=bool(torch.equal(ref, outd[:m[2] * R])))
