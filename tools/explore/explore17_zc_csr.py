"""Zero-copy CSR (NEXT-3): sampler time per minibatch with the CSR in HBM vs left in pinned host
memory, whole GPU and on an 8-SM green-context partition; configs 3 and 4.
    python tools/explore17_zc_csr.py > gpurun_out/explore17_zc_csr.jsonl"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
for cid in (3, 4):
    c = gen.CONFIGS[cid]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    graphs = {"hbm": dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda()),
              "host cols (offsets in HBM)": dgz.HostGraph(off, col),
              "host cols + offsets": dgz.HostGraph(off, col, offsets_in_hbm=False)}
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts)
    seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(24)]
    rs = [gen.batch_rng_seed(c.seed, j) for j in range(24)]
    part = dgz.Partition(8, -1, dgz.PARTITION_SPREAD)
    for where, g in graphs.items():
        for sname, stream in (("whole GPU", torch.cuda.Stream()), ("8-SM partition", part.fetch_stream)):
            for j in range(4):
                dgz.sample_uniform(g, seeds[j], c.fanouts, rs[j], bufs, stream=stream)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ms = []
            for j in range(4, 24):
                a.record(stream)
                dgz.sample_uniform(g, seeds[j], c.fanouts, rs[j], bufs, stream=stream)
                b.record(stream)
                b.synchronize()
                ms.append(a.elapsed_time(b))
            print(json.dumps({"config": cid, "csr": where, "where": sname, "sample_ms_p50": round(float(np.median(ms)), 4),
                              "sample_ms_p90": round(float(np.percentile(ms, 90)), 4),
                              "rows": int(bufs.sizes_host[-1])}), flush=True)
    torch.cuda.synchronize()
    part.destroy()
    for k in list(graphs)[1:]:
        graphs[k].close()
    del graphs, bufs
