"""Diagnose slow "fetch alone" timings on partitions: per-fetch time (host-synchronised, as the
training example measures it) with the partition gather config with / without the work counter,
sampler on the compute stream, config 3.
    python tools/explore32_fetch_alone.py"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402
from paper_2103_03330_b200.pipeline import MinibatchFetcher  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[3]
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(12)]
rs = [gen.batch_rng_seed(c.seed, j) for j in range(12)]
part = dgz.Partition(16, -1, 0)
for name, flags, sample_on_comp in (("static", dgz.FLAG_DEEP, True), ("dynamic", dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC, True),
                                    ("dynamic, sampler on fetch", dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC, False)):
    cfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=8, flags=flags)
    f = MinibatchFetcher(table, graph, c.fanouts, c.batch, fetch_stream=part.fetch_stream, gather_cfg=cfg,
                         sample_stream=part.compute_stream if sample_on_comp else None)
    for i in range(2):
        f.fetch(seeds[i], rs[i]).sizes()
    torch.cuda.synchronize()
    ts = []
    for i in range(2, 12):
        t0 = time.perf_counter()
        mb = f.fetch(seeds[i], rs[i], timing=True)
        mb.sizes()
        ts.append((time.perf_counter() - t0) * 1e3)
        gt = mb.timing[1].elapsed_time(mb.timing[2])
    print(json.dumps({"arm": name, "host_ms_per_fetch": [round(x, 2) for x in ts], "last_gather_ms": round(gt, 3)}), flush=True)
    f.close()
    del f
part.destroy()
table.unregister()
buf.free()
