"""ncu evidence for the HBM hot-row cache (NEXT-1): one config-4 minibatch of the power-law graph
gathered through a 20 % cache; the cached gather should read over PCIe exactly the sectors of the
rows that missed the cache.  Writes the expected counts next to the capture.
    ncu -k regex:gather_segment_kernel -s 1 -c 1 --metrics ... python tools/cache_ncu.py out.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed, skew_alpha=3.0)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
order = torch.argsort(torch.bincount(g.cols.long(), minlength=c.n_nodes), descending=True)
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
dgz.sample_uniform(g, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, 0)).cuda(), c.fanouts,
                   gen.batch_rng_seed(c.seed, 0), bufs)
torch.cuda.synchronize()
n = int(bufs.sizes_host[-1])
ids, pos = bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone()
k = int(c.n_nodes * 0.20)
cache = dgz.HotRowCache(tb, order[:k].contiguous())              # launch 1 of the gather kernel: the fill
out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
cache.gather(ids, out, dst_pos=pos, n=n)                          # launch 2: the cached gather (profiled)
torch.cuda.synchronize()
miss = int((cache.slot_map[ids] < 0).sum())
with open(sys.argv[1], "w") as f:
    json.dump({"rows": n, "row_bytes": R, "cache_fraction": 0.20, "missed_rows": miss, "hit_rows": n - miss,
               "expected_sysmem_sectors_if_unmerged": miss * (R // 32)}, f)
tb.unregister()
buf.free()
