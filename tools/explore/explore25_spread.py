"""Is the translation-bound gather limited per GPC?  The sorted config-4 gather alone on a green-context
partition of k SMs taken across every GPC (DGZ_PARTITION_SPREAD) vs k contiguous SMs (the split's
first groups), one 8-warp CTA per SM, 16 loads per lane, eight fresh minibatches.
    python tools/explore25_spread.py > gpurun_out/explore25_spread.jsonl"""
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
for rep in range(2):
    for k in (8, 16, 24, 32, 48):
        for spread in (True, False):
            part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD if spread else 0)
            for w in (4, 8):
                for sb in sbs:   # fresh minibatches for every measurement
                    dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(),
                                       c.fanouts, gen.batch_rng_seed(c.seed, j), sb)
                    j += 1
                torch.cuda.synchronize()
                nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
                cfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=w, flags=dgz.FLAG_DEEP)
                s = part.fetch_stream
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for sb in sbs:
                    dgz.gather_perm(table, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1],
                                    n_dev=sb.sizes_dev[L:L + 1], cfg=cfg, stream=s)
                b.record(s)
                torch.cuda.synchronize()
                print(json.dumps({"rep": rep, "sms": part.fetch_sms, "spread": spread, "warps": w,
                                  "gbs": round(nrows * c.row_bytes / a.elapsed_time(b) / 1e6, 2)}), flush=True)
            part.destroy()
table.unregister()
buf.free()
