"""Sorted (sampler-order) rows: does a narrow in-flight window beat the translation limit?"""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz

def out(**kw): print(json.dumps(kw), flush=True)

def ev_time(fn, iters=3, warm=1):
    for _ in range(warm): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
total = c.table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, 0)).cuda()
dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, 0), bufs)
torch.cuda.synchronize()
n = int(bufs.sizes_host[-1])
U = bufs.ids[:n].clone()
Us = torch.sort(U).values
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
for name, ids in (("sampler_order", U), ("fully_sorted", Us)):
    for variant in (1, 4):
        for sms in (1, 2, 4, 8, 16, 32, 64, 148):
            for warps in ((4, 8, 16, 32) if variant == 1 else (4, 8, 32)):
                cfg = dgz.gather_cfg(variant=variant, sm_count=sms, warps_per_cta=warps)
                tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n, cfg=cfg))
                out(order=name, variant=variant, sms=sms, warps=warps, gbs=n * R / tt / 1e9)
