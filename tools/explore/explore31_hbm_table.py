"""All-in-GPU reference: the 56.9 GB config-4 table copied into HBM and gathered by the same
kernels -- launch shapes and variants (SEGMENT 8/16 loads per lane, warps x CTAs, BULK/TMA),
sorted (gather_perm) vs frontier order (gather), eight config-4 minibatches.
    python tools/explore31_hbm_table.py > gpurun_out/explore31_hbm_table.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
L = len(c.fanouts)
host = torch.empty(c.table_bytes, dtype=torch.uint8)
gen.fill_table(host.data_ptr(), c.table_bytes, c.seed)
dev = host.cuda()
del host
dt = dgz.DeviceTable(dev.data_ptr(), c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
sbs = []
for j in range(8):
    sb = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False)
    dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                       gen.batch_rng_seed(c.seed, j), sb)
    sbs.append(sb)
torch.cuda.synchronize()
nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
out = torch.empty(sbs[0].bounds[-1] * R, dtype=torch.uint8, device="cuda")
ARMS = {"default": None,
        "16 warps x 4, deep": dgz.gather_cfg(warps_per_cta=16, ctas_per_sm=4, flags=dgz.FLAG_DEEP),
        "8 warps x 8": dgz.gather_cfg(warps_per_cta=8, ctas_per_sm=8),
        "8 warps x 8, deep": dgz.gather_cfg(warps_per_cta=8, ctas_per_sm=8, flags=dgz.FLAG_DEEP),
        "16 warps x 2": dgz.gather_cfg(warps_per_cta=16, ctas_per_sm=2),
        "bulk 8 warps": dgz.gather_cfg(variant=dgz.GATHER_BULK),
        "bulk 16 warps x 2": dgz.gather_cfg(variant=dgz.GATHER_BULK, warps_per_cta=16, ctas_per_sm=2)}
for order in ("sorted", "frontier"):
    for name, cfg in ARMS.items():
        def run():
            for sb in sbs:
                if order == "sorted":
                    dgz.gather_perm(dt, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1], n_dev=sb.sizes_dev[L:L + 1],
                                    cfg=cfg)
                else:
                    dgz.gather(dt, sb.ids, out, n=sb.bounds[-1], n_dev=sb.sizes_dev[L:L + 1], cfg=cfg or dgz.gather_cfg())
        run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        useful = nrows * R / ms / 1e6
        print(json.dumps({"order": order, "arm": name, "useful_gbs": round(useful, 1),
                          "hbm_traffic_gbs": round(useful * 2 + nrows * 16 / ms / 1e6, 1)}), flush=True)
dt.unregister()
