"""A/B on one box: line merging (default) vs NO_MERGE for configs 3 and 4 (sampler output)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
for cid in (3, 4):
    c = gen.CONFIGS[cid]; R = c.row_bytes
    buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
    mbs = []
    for j in range(6):
        seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda()
        dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, j), bufs); torch.cuda.synchronize()
        n = int(bufs.sizes_host[-1]); mbs.append((bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone(), n))
    outd = torch.empty(max(m[2] for m in mbs) * R, dtype=torch.uint8, device="cuda")
    res = {0: [], 1: []}
    for rep in range(4):
        for flags in (0, 1):
            cfg = dgz.gather_cfg(flags=flags) if flags else None
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            for m in mbs: dgz.gather_perm(tb, m[0], m[1], outd, n=m[2], cfg=cfg)
            b.record(); torch.cuda.synchronize()
            res[flags].append(sum(m[2] for m in mbs) * R / (a.elapsed_time(b) * 1e6))
    print(json.dumps({"config": cid, "merge_gbs": [round(x, 2) for x in res[0]], "no_merge_gbs": [round(x, 2) for x in res[1]]}), flush=True)
    tb.unregister(); buf.free(); del g, bufs, mbs, outd; torch.cuda.empty_cache()
