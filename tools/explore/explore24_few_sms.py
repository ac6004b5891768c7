"""How few SMs can carry the sorted config-4 gather?  SEGMENT (LDG, 16 loads per lane, 8 or 16 warps
per CTA) vs BULK (one cp.async.bulk / TMA op per row into a shared-memory ring) on k = 2..32 SMs,
bounded grids on the whole GPU (no co-runner), eight fresh config-4 minibatches.
    python tools/explore24_few_sms.py > gpurun_out/explore24_few_sms.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
sbs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False) for _ in range(8)]
out = torch.empty(sbs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
j = 0
ARMS = [("segment", dgz.GATHER_SEGMENT, 8, dgz.FLAG_DEEP), ("segment", dgz.GATHER_SEGMENT, 16, dgz.FLAG_DEEP),
        ("bulk", dgz.GATHER_BULK, 8, 0), ("bulk", dgz.GATHER_BULK, 16, 0)]
for k in (2, 4, 8, 16, 32):
    for name, v, w, fl in ARMS:
        for sb in sbs:
            dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                               gen.batch_rng_seed(c.seed, j), sb)
            j += 1
        torch.cuda.synchronize()
        nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
        cfg = dgz.gather_cfg(variant=v, sm_count=k, warps_per_cta=w, flags=fl)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for sb in sbs:
            dgz.gather_perm(table, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1], n_dev=sb.sizes_dev[L:L + 1], cfg=cfg)
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"sms": k, "variant": name, "warps": w, "gbs": round(nrows * c.row_bytes / a.elapsed_time(b) / 1e6, 2)}),
              flush=True)
table.unregister()
buf.free()
