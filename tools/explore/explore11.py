"""Hide the sampler behind the previous gather: sampler on a small green-context partition."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
from paper_2103_03330_b200.pipeline import MinibatchFetcher

def out(**kw): print(json.dumps(kw), flush=True)
torch.cuda.set_device(0)
c = gen.CONFIGS[4]; R = c.row_bytes; L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
K = 30
seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(K + 3)]
rng = [gen.batch_rng_seed(c.seed, j) for j in range(K + 3)]
ns = torch.zeros(K + 3, dtype=torch.int64, device="cuda")
def run(f, name):
    for i in range(3): f.fetch(seeds[i], rng[i])
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(f.sample_stream)
    for i in range(3, K + 3): f.fetch(seeds[i], rng[i], count_into=ns[i:i + 1])
    f.stream.wait_stream(f.sample_stream); b.record(f.stream); torch.cuda.synchronize()
    t = a.elapsed_time(b) / K
    out(mode=name, ms_per_step=round(t, 3), gbs=round(float(ns[3:].float().mean()) * R / t / 1e6, 2))
run(MinibatchFetcher(tb, g, c.fanouts, c.batch), "sequential")
run(MinibatchFetcher(tb, g, c.fanouts, c.batch, overlap_sampling=True), "two_streams_full_gpu")
for k in (8, 16, 32):
    part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD)
    f = MinibatchFetcher(tb, g, c.fanouts, c.batch, sample_stream=part.fetch_stream)
    run(f, f"sampler_on_{part.fetch_sms}_sm_partition")
    del f; torch.cuda.synchronize(); part.destroy()
    part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD)
    f = MinibatchFetcher(tb, g, c.fanouts, c.batch, sample_stream=part.fetch_stream, fetch_stream=part.compute_stream)
    f.sample_stream = part.fetch_stream
    run(f, f"sampler_on_{part.fetch_sms}_gather_on_{part.compute_sms}")
    del f; torch.cuda.synchronize(); part.destroy()
