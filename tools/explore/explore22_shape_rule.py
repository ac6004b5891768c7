"""A/B of the sorted gather's launch-shape rule (rows in flight sized by row width and sparsity) against
the previous fixed default (148 CTAs x 2 warps, 16 loads per lane), on FRESH lists every repetition
(no L2-resident page-table lines from a previous pass): 256 MiB and 64 MiB of sorted random distinct
rows per width over the 56.9 GB buffer, and eight config-4 minibatches.
    python tools/explore22_shape_rule.py > gpurun_out/explore22_shape_rule.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
total = c.table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, c.seed)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ARMS = {"old_default_148x2": dgz.gather_cfg(sm_count=148, warps_per_cta=2, flags=dgz.FLAG_DEEP), "rule": None,
        "37x1": dgz.gather_cfg(sm_count=37, warps_per_cta=1, flags=dgz.FLAG_DEEP),
        "74x1": dgz.gather_cfg(sm_count=74, warps_per_cta=1, flags=dgz.FLAG_DEEP),
        "148x1": dgz.gather_cfg(sm_count=148, warps_per_cta=1, flags=dgz.FLAG_DEEP)}


def run_lists(tb, lists, n, cfg, ns=None):
    torch.cuda.synchronize()
    a.record()
    for i, (srt, pos) in enumerate(lists):
        dgz.gather_perm(tb, srt, pos, outd, n=n, n_dev=None if ns is None else ns[i], cfg=cfg)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
for R in (16, 64, 128, 256, 400, 512, 1024, 2408):
    rows = total // R
    tb = dgz.register_table(buf.ptr, rows, R // 4 if R % 4 == 0 else R, dgz.F32 if R % 4 == 0 else dgz.U8)
    for mib in (64, 256):
        n = (mib << 20) // R
        seed = 0
        for arm, cfg in ARMS.items():
            ms_tot, cnt = 0.0, 0
            for rep in range(2):
                lists = []
                for _ in range(3):
                    seed += 1
                    lists.append(dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 1000 + mib * 10 + seed)).cuda(), rows))
                ms = run_lists(tb, lists, n, cfg)
                if rep:
                    ms_tot += ms
                    cnt += 3
                del lists
            print(json.dumps({"R": R, "mib": mib, "gap_kb": round(total / n / 1024, 1), "arm": arm,
                              "gbs": round(cnt * n * R / ms_tot / 1e6, 2)}), flush=True)
    tb.unregister()
del outd

table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
L = len(c.fanouts)
sbs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False, sorted_ids=True) for _ in range(8)]
outd = torch.empty(sbs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
j = 0
for rep in range(2):
    for arm, cfg in ARMS.items():
        for sb in sbs:
            dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                               gen.batch_rng_seed(c.seed, j), sb)
            j += 1
        torch.cuda.synchronize()
        nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
        ms = run_lists(table, [(sb.ids_sorted, sb.ids_sorted_pos) for sb in sbs], sbs[0].bounds[-1], cfg,
                       ns=[sb.sizes_dev[L:L + 1] for sb in sbs])
        print(json.dumps({"R": 512, "case": "config4 minibatches (fresh)", "rep": rep, "arm": arm,
                          "gbs": round(nrows * c.row_bytes / ms / 1e6, 2)}), flush=True)
table.unregister()
buf.free()
