"""L2 cache hints on the product gather: do evict-first stores / loads keep the GPU page-table
lines (walked for every zero-copy translation miss) resident and raise the translation-bound rate?
Config-4 minibatches (sampler -> sorted gather) and 256 MiB of sorted random rows at 128 / 512 B.
    python tools/explore18_cache_hints.py > gpurun_out/explore18_cache_hints.jsonl"""
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
FLAGS = {"none": 0, "cs_stores": dgz.FLAG_STREAM_STORES, "ef_loads": dgz.FLAG_EVICT_FIRST_LOADS,
         "both": dgz.FLAG_STREAM_STORES | dgz.FLAG_EVICT_FIRST_LOADS}
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


# config-4 minibatches: 8 different sampled minibatches, gathered in turn
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
    for name, fl in FLAGS.items():
        cfg = dgz.gather_cfg(flags=fl)

        def run():
            for m in mbs:
                dgz.gather_perm(table, m.ids_sorted, m.ids_sorted_pos, out, n=m.bounds[-1], n_dev=m.sizes_dev[L:L + 1], cfg=cfg)
        ms = timeit(run, 2)
        print(json.dumps({"case": "config4 minibatches", "hints": name, "rep": rep,
                          "gbs": round(nrows * c.row_bytes / (ms * 1e-3) / 1e9, 2)}), flush=True)
table.unregister()
del mbs, graph, out

outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
for R in (128, 512):
    rows = c.table_bytes // R
    n = (256 << 20) // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    lists = []
    for s in range(3):
        ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 11 + s)).cuda()
        lists.append(dgz.order_ids(ids, rows))
    for name, fl in FLAGS.items():
        cfg = dgz.gather_cfg(flags=fl)

        def run():
            for srt, pos in lists:
                dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
        ms = timeit(run, 2)
        print(json.dumps({"case": f"sorted random rows R={R}", "hints": name, "gbs": round(3 * n * R / (ms * 1e-3) / 1e9, 2)}),
              flush=True)
    tb.unregister()
buf.free()
