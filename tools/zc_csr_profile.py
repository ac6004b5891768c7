"""One config-4 minibatch sampled from a zero-copy CSR (dgz.HostGraph), for ncu: how many sysmem
requests / sectors does each hop's sampling kernel issue, vs frontier nodes and sampled slots?
    ncu -k regex:hop_sample --metrics ... python tools/zc_csr_profile.py"""
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
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.HostGraph(off, col)
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts)
seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, 3)).cuda()
dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, 3), bufs)
torch.cuda.synchronize()
sizes = bufs.sizes_host.tolist()
ids = bufs.ids[:sizes[-1]].cpu().numpy()
rec = {"sizes": sizes, "hops": []}
for k, f in enumerate(c.fanouts):
    fr = ids[:sizes[k]]
    deg = off[fr + 1] - off[fr]
    slots = np.minimum(deg, f)
    rec["hops"].append({"k": k, "nodes": int(sizes[k]), "slots": int(slots.sum()),
                        "adjacency_sectors_touched_max": int(sum(((off[fr] + deg) * 4 + 31) // 32 - (off[fr] * 4) // 32))})
print(json.dumps(rec))
g.close()
