"""In-flight window of the sorted zero-copy gather, finer: CTAs x warps x loads per lane for config-4
minibatches and 256 MiB of sorted random rows at R = 128 / 256 / 512 / 2048 B.
    python tools/explore20_inflight.py > gpurun_out/explore20_inflight.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
SHAPES = [(0, 0, 0), (148, 2, 2), (148, 1, 2), (148, 1, 0), (120, 1, 2), (96, 1, 2), (74, 1, 2), (74, 2, 2), (48, 2, 2),
          (148, 3, 2), (148, 4, 0)]


def timeit(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
mbs = []
for j in range(8):
    sb = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False, sorted_ids=True)
    dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                       gen.batch_rng_seed(c.seed, j), sb)
    mbs.append(sb)
torch.cuda.synchronize()
out = torch.empty(mbs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
L = len(c.fanouts)
nrows = sum(int(m.sizes_host[-1]) for m in mbs)
for rep in range(2):
    for sms, warps, flags in SHAPES:
        cfg = dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, flags=flags)

        def run():
            for m in mbs:
                dgz.gather_perm(table, m.ids_sorted, m.ids_sorted_pos, out, n=m.bounds[-1], n_dev=m.sizes_dev[L:L + 1], cfg=cfg)
        ms = timeit(run)
        print(json.dumps({"case": "config4", "rep": rep, "sms": sms, "warps": warps, "deep": flags == 2,
                          "gbs": round(nrows * c.row_bytes / (ms * 1e-3) / 1e9, 2)}), flush=True)
table.unregister()
del mbs, graph, out

outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
for R in (128, 256, 512, 2048):
    rows = c.table_bytes // R
    n = (256 << 20) // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    srt, pos = dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 17)).cuda(), rows)
    for sms, warps, flags in SHAPES:
        cfg = dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, flags=flags)
        ms = timeit(lambda: dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg), 3)
        print(json.dumps({"case": f"R={R}", "sms": sms, "warps": warps, "deep": flags == 2, "gbs": round(n * R / ms / 1e6, 2)}),
              flush=True)
    tb.unregister()
buf.free()
