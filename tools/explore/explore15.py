"""Per-SM fetch throughput on small green-context partitions: schedule x warps x depth."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
def out(**kw): print(json.dumps(kw), flush=True)
torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, 0)).cuda()
dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, 0), bufs); torch.cuda.synchronize()
n = int(bufs.sizes_host[-1]); ids = bufs.ids_sorted[:n].clone(); pos = bufs.ids_sorted_pos[:n].clone()
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
for k in (8, 16):
    part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD)
    s = part.fetch_stream
    for sched in (1, 2):
        for ctas, warps, flags in ((k, 2, 2), (k, 8, 2), (k, 16, 0), (2 * k, 8, 2), (4 * k, 4, 2), (148, 2, 2)):
            cfg = dgz.gather_cfg(sm_count=ctas, warps_per_cta=warps, flags=flags, schedule=sched)
            for _ in range(2): dgz.gather_perm(tb, ids, pos, outd, n=n, cfg=cfg, stream=s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record(s)
            for _ in range(3): dgz.gather_perm(tb, ids, pos, outd, n=n, cfg=cfg, stream=s)
            b.record(s); torch.cuda.synchronize()
            t = a.elapsed_time(b) / 3
            out(part_sms=part.fetch_sms, sched=sched, ctas=ctas, warps=warps, flags=flags, gbs=round(n * R / t / 1e6, 2))
    part.destroy()
