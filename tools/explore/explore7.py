"""Sorted gather: cache-policy hints x loads in flight x grid shape (config-4 sampler output)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz

def out(**kw): print(json.dumps(kw), flush=True)
def ev_time(fn, iters=4, warm=1):
    for _ in range(warm): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters

torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
ids_l, pos_l, ns = [], [], []
for j in range(4):
    seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda()
    dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, j), bufs)
    torch.cuda.synchronize()
    n = int(bufs.sizes_host[-1]); ns.append(n)
    ids_l.append(bufs.ids_sorted[:n].clone()); pos_l.append(bufs.ids_sorted_pos[:n].clone())
outd = torch.empty(max(ns) * R, dtype=torch.uint8, device="cuda")
it = [0]
def run(cfg):
    def f():
        k = it[0] % 4; it[0] += 1
        dgz.gather_perm(tb, ids_l[k], pos_l[k], outd, n=ns[k], cfg=cfg)
    return f
nmean = sum(ns) / 4
for flags in (0, 1, 2, 3):
    for sms, warps in ((48, 2), (64, 2), (96, 1), (96, 2), (148, 1), (148, 2), (74, 4), (32, 4), (24, 4), (16, 8)):
        cfg = dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, flags=flags)
        tt = ev_time(run(cfg))
        out(flags=flags, sms=sms, warps=warps, gbs=round(nmean * R / tt / 1e9, 2))
