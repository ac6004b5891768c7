"""Default pipeline (sampler on an 8-SM partition, gather on the other 140): does sizing the gather
grid to the 140 SMs it actually has (instead of 148 CTAs, 8 SMs doubled up) or the work-counter
schedule change the step throughput?  40 fresh config-4 minibatches per arm, two reps.
    python tools/explore29_pipeline_grid.py > gpurun_out/explore29_pipeline_grid.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402
from paper_2103_03330_b200.pipeline import MinibatchFetcher  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
K = 40
ARMS = {"default (148 CTAs x 2 warps, static)": None,
        "140 CTAs x 2 warps, static": dgz.gather_cfg(sm_count=140, warps_per_cta=2, flags=dgz.FLAG_DEEP),
        "148 CTAs x 2 warps, work counter": dgz.gather_cfg(flags=dgz.FLAG_DYNAMIC),
        "140 CTAs x 2 warps, work counter": dgz.gather_cfg(sm_count=140, warps_per_cta=2,
                                                           flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)}
j = 0
for rep in range(2):
    for name, cfg in ARMS.items():
        f = MinibatchFetcher(table, graph, c.fanouts, c.batch, gather_cfg=cfg)
        seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j + i)).cuda() for i in range(K + 3)]
        rs = [gen.batch_rng_seed(c.seed, j + i) for i in range(K + 3)]
        j += K + 3
        cnt = torch.zeros(K, dtype=torch.int64, device="cuda")
        for i in range(3):
            f.fetch(seeds[i], rs[i])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(f.sample_stream)
        for i in range(K):
            f.fetch(seeds[3 + i], rs[3 + i], count_into=cnt[i:i + 1])
        f.stream.wait_stream(f.sample_stream)
        b.record(f.stream)
        torch.cuda.synchronize()
        gbs = float(cnt.sum()) * R / (a.elapsed_time(b) * 1e-3) / 1e9
        print(json.dumps({"rep": rep, "arm": name, "step_gbs": round(gbs, 2)}), flush=True)
        f.close()
        del f
table.unregister()
buf.free()
