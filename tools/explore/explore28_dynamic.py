"""A/B: static interleaved batch schedule vs a work counter (DGZ_GATHER_FLAG_DYNAMIC) for the sorted
gather -- whole GPU (default launch shape) and green-context partitions -- on fresh config-4
minibatches and fresh 256 MiB lists of sorted random rows (R = 128 / 256 / 512 B).
    python tools/explore28_dynamic.py > gpurun_out/explore28_dynamic.jsonl"""
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
sbs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False) for _ in range(6)]
out = torch.empty(sbs[0].bounds[-1] * c.row_bytes + (256 << 20), dtype=torch.uint8, device="cuda")
j = [0]
parts = {"whole GPU": None, "16 contiguous": dict(sms=16, flags=0), "16 spread": dict(sms=16, flags=dgz.PARTITION_SPREAD),
         "24 spread": dict(sms=24, flags=dgz.PARTITION_SPREAD)}


def timed(s, fn):
    fn()   # warm-up
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for rep in range(2):
    for pname, pdesc in parts.items():
        part = dgz.Partition(pdesc["sms"], -1, pdesc["flags"]) if pdesc else None
        s = part.fetch_stream if part else torch.cuda.current_stream()
        for dyn in (False, True):
            fl = dgz.FLAG_DYNAMIC if dyn else 0
            cfg = (dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=8, flags=dgz.FLAG_DEEP | fl) if part
                   else dgz.gather_cfg(flags=fl))
            for sb in sbs:
                dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j[0])).cuda(),
                                   c.fanouts, gen.batch_rng_seed(c.seed, j[0]), sb)
                j[0] += 1
            torch.cuda.synchronize()
            nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)

            def run():
                for sb in sbs:
                    dgz.gather_perm(table, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1],
                                    n_dev=sb.sizes_dev[L:L + 1], cfg=cfg, stream=s)
            ms = timed(s, run) / 1.0
            print(json.dumps({"rep": rep, "case": "config4", "where": pname, "dynamic": dyn,
                              "gbs": round(nrows * c.row_bytes / ms / 1e6, 2)}), flush=True)
        if part:
            part.destroy()
table.unregister()
for R in (128, 256, 512):
    rows = c.table_bytes // R
    n = (256 << 20) // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    for rep in range(2):
        for dyn in (False, True):
            j[0] += 1
            srt, pos = dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 100 + j[0])).cuda(), rows)
            cfg = dgz.gather_cfg(flags=dgz.FLAG_DYNAMIC if dyn else 0)
            s = torch.cuda.current_stream()
            ms = timed(s, lambda: dgz.gather_perm(tb, srt, pos, out, n=n, cfg=cfg))
            print(json.dumps({"rep": rep, "case": f"R={R}", "where": "whole GPU", "dynamic": dyn,
                              "gbs": round(n * R / ms / 1e6, 2)}), flush=True)
    tb.unregister()
buf.free()
