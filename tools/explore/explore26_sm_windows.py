"""Which SMs walk fastest?  The sorted config-4 gather alone on a green-context partition made of an
explicit window of minimal SM groups (dgz_partition_create_groups): windows of W groups at every
offset of the driver's group order, plus strided picks; eight fresh minibatches per point.
    python tools/explore26_sm_windows.py > gpurun_out/explore26_sm_windows.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
ng, per = dgz.partition_groups()
print(json.dumps({"groups": ng, "sms_per_group": per}), flush=True)
c = gen.CONFIGS[4]
L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
sbs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False) for _ in range(6)]
out = torch.empty(sbs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
j = 0


def run(groups, label):
    global j
    part = dgz.Partition(0, -1, groups=groups)
    for sb in sbs:
        dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                           gen.batch_rng_seed(c.seed, j), sb)
        j += 1
    torch.cuda.synchronize()
    nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
    cfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=8, flags=dgz.FLAG_DEEP)
    s = part.fetch_stream
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for sb in sbs:
        dgz.gather_perm(table, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1], n_dev=sb.sizes_dev[L:L + 1], cfg=cfg,
                        stream=s)
    b.record(s)
    torch.cuda.synchronize()
    print(json.dumps({"pick": label, "groups": groups, "sms": part.fetch_sms,
                      "gbs": round(nrows * c.row_bytes / a.elapsed_time(b) / 1e6, 2)}), flush=True)
    part.destroy()


W = max(1, 16 // per)
for o in range(0, ng - W + 1, W):
    run(list(range(o, o + W)), f"window {W} groups at {o}")
for stride in (2, 4, 8, 9):
    g = list(range(0, ng, stride))[:W]
    if len(g) == W:
        run(g, f"stride {stride}")
table.unregister()
buf.free()
