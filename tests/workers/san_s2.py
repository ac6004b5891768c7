"""compute-sanitizer target (test infrastructure: it checks against the oracle) for the session-2 features (tools/sanitize_s2.sh): zero-copy CSR
sampling, the sorted gather's default launch shapes, cache hints, local-shard cache fill + cached
gather, order_ids -- each checked against the oracle so a silent corruption also fails."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
import oracle  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[1]
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, 1)
rs = gen.batch_rng_seed(c.seed, 1)
want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs)
g = dgz.HostGraph(off, col)
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts)
dgz.sample_uniform(g, torch.from_numpy(seeds).cuda(), c.fanouts, rs, bufs)
torch.cuda.synchronize()
assert np.array_equal(bufs.ids[:bufs.sizes_host[-1]].cpu().numpy(), want.U)
g.close()
for R, rows, n, flags in ((128, 400_000, 1500, 0), (128, 40_000, 6000, 0), (400, 20_000, 4000, 0), (1028, 6000, 1500, 24)):
    buf = dgz.HostBuffer(rows * R + 8192)
    gen.fill_table(buf.ptr + 4, rows * R, R)
    t = dgz.register_table(buf.ptr + 4, rows, R // 4, dgz.F32)
    host = buf.numpy(4, rows * R)
    idx = gen.random_ids(rows, n, R)
    exp, _ = oracle.gather(host, R, idx)
    srt, pos = dgz.order_ids(torch.from_numpy(idx).cuda(), rows)
    out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
    dgz.gather_perm(t, srt, pos, out, cfg=dgz.gather_cfg(flags=flags) if flags else None)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(n, R), exp), (R, n)
    hot = torch.from_numpy(gen.distinct_ids(rows, rows // 5, 3)).cuda()
    cache = dgz.HotRowCache(t, hot, n_shards=2)
    cache.gather(srt, out, dst_pos=pos)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(n, R), exp), ("cached", R, n)
    del cache
    t.unregister()
    buf.free()
print("session-2 paths ok")
