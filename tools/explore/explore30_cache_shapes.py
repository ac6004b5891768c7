"""NEXT-1 cached gather: launch shapes.  Power-law config-4 graph (alpha 3), top 5 / 20 % of rows by
in-degree cached in HBM, eight sampled minibatches gathered in address order with
dgz_gather_cached: default shape vs 1 warp per SM, half the SMs, and the work-counter schedule.
    python tools/explore30_cache_shapes.py > gpurun_out/explore30_cache_shapes.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed, skew_alpha=3.0)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
order = torch.argsort(torch.bincount(g.cols.long(), minlength=c.n_nodes), descending=True)
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
mbs = []
for j in range(8):
    dgz.sample_uniform(g, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                       gen.batch_rng_seed(c.seed, j), bufs)
    torch.cuda.synchronize()
    n = int(bufs.sizes_host[-1])
    mbs.append((bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone(), n))
nrows = sum(m[2] for m in mbs)
outd = torch.empty(max(m[2] for m in mbs) * R, dtype=torch.uint8, device="cuda")
nsm = dgz.device_sm_count()
SHAPES = {"default (148 x 2, 16 loads)": None,
          "148 x 1": dgz.gather_cfg(sm_count=nsm, warps_per_cta=1, flags=dgz.FLAG_DEEP),
          "74 x 2": dgz.gather_cfg(sm_count=nsm // 2, warps_per_cta=2, flags=dgz.FLAG_DEEP),
          "148 x 4": dgz.gather_cfg(sm_count=nsm, warps_per_cta=4, flags=dgz.FLAG_DEEP),
          "148 x 2, work counter": dgz.gather_cfg(flags=dgz.FLAG_DYNAMIC)}
for frac in (0.05, 0.20):
    k = int(c.n_nodes * frac)
    cache = dgz.HotRowCache(tb, order[:k].contiguous())
    torch.cuda.synchronize()
    hit = float(np.mean([float((cache.slot_map[m[0]] >= 0).float().mean()) for m in mbs]))
    for rep in range(2):
        for name, cfg in SHAPES.items():
            for m in mbs[:2]:
                cache.gather(m[0], outd, dst_pos=m[1], n=m[2], cfg=cfg)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for m in mbs:
                cache.gather(m[0], outd, dst_pos=m[1], n=m[2], cfg=cfg)
            b.record()
            torch.cuda.synchronize()
            print(json.dumps({"cache_frac": frac, "hit_rate": round(hit, 4), "rep": rep, "shape": name,
                              "effective_gbs": round(nrows * R / a.elapsed_time(b) / 1e6, 2)}), flush=True)
    del cache
    torch.cuda.empty_cache()
tb.unregister()
buf.free()
