"""NEXT-1 cached gather on a managed host table: launch shape (warps per SM) with 20 % of the rows of
the power-law config-4 graph cached in HBM; eight sampled minibatches gathered in address order.
The registered-table default (one warp per SM) was chosen because the missed rows are the sparse,
page-walk-bound part of the list; without walks (managed table) more rows in flight may pay.

    python tools/cache_managed_shapes.py > gpurun_out/cache_managed_shapes.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
for kind in ("managed", "registered"):
    buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_MANAGED if kind == "managed" else dgz.HOST_HUGEPAGE)
    gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed, skew_alpha=3.0)
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    del off, col
    order = torch.argsort(torch.bincount(g.cols.long(), minlength=c.n_nodes), descending=True)
    cache = dgz.HotRowCache(tb, order[:int(0.2 * c.n_nodes)].contiguous(), 1)
    del order
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False)
    mbs = []
    for j in range(8):
        dgz.sample_uniform(g, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                           gen.batch_rng_seed(c.seed, j), bufs)
        torch.cuda.synchronize()
        n = int(bufs.sizes_host[-1])
        mbs.append((bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone(), n))
    out = torch.empty(max(m[2] for m in mbs) * R, dtype=torch.uint8, device="cuda")
    rows = sum(m[2] for m in mbs)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for shape in (None, (1, 2), (2, 2), (4, 2), (8, 2)):
        cfg = None if shape is None else dgz.gather_cfg(sm_count=148, warps_per_cta=shape[0], flags=shape[1])
        for m in mbs[:2]:
            cache.gather(m[0], out, dst_pos=m[1], n=m[2], cfg=cfg)
        torch.cuda.synchronize()
        a.record()
        for m in mbs:
            cache.gather(m[0], out, dst_pos=m[1], n=m[2], cfg=cfg)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"table": kind, "shape": "default" if shape is None else list(shape),
                          "effective_gbs": round(rows * R / (a.elapsed_time(b) * 1e-3) / 1e9, 2)}), flush=True)
    del cache, g
    tb.unregister()
    buf.free()
    torch.cuda.empty_cache()
