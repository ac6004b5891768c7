"""NEXT-1 on N GPUs: the HBM hot-row cache SHARDED across the ranks (dgz.ShardedHotRowCache: rank g
holds hot rows g, g + G, ... in its HBM; the others read them by NVLink peer loads through CUDA IPC
mappings), on the power-law papers100M-shaped graph.  One process per GPU:

    torchrun --nproc-per-node N tools/cache_sharded_experiment.py [alpha] [frac ...]

Each rank fetches its own minibatches (global batch j = i*G + rank) uncached and cached, and rank 0
prints per-rank and aggregate GB/s, the hit rate and the share of hits served by peer GPUs.  On a
one-GPU box (DGZ_BENCH_SAME_DEVICE=1, gloo) every "peer" shard is local HBM: the run validates
the code path, not NVLink bandwidth.
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


def main():
    same = os.environ.get("DGZ_BENCH_SAME_DEVICE") == "1"
    dist.init_process_group("gloo" if same else "nccl")
    G, rank = dist.get_world_size(), dist.get_rank()
    dev = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    bar = (lambda: dist.barrier()) if same else (lambda: dist.barrier(device_ids=[dev]))
    alpha = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
    fracs = [float(x) for x in sys.argv[2:]] or [0.05, 0.20]
    c = gen.CONFIGS[4]
    R = c.row_bytes
    name = f"/dgz_cache_exp_{os.environ.get('MASTER_PORT', '0')}"
    gen.set_threads(max(1, (os.cpu_count() or 1) // G))
    if rank == 0:
        buf = dgz.HostBuffer(c.table_bytes + 4096, shm_name=name, create=True)
        gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    bar()
    if rank != 0:
        buf = dgz.HostBuffer(c.table_bytes + 4096, shm_name=name, create=False)
    bar()
    if rank == 0:
        buf.unlink()
    tb = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed, skew_alpha=alpha)
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    del off, col
    order = torch.argsort(torch.bincount(g.cols.long(), minlength=c.n_nodes), descending=True)
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
    mbs = []
    for i in range(8):
        j = i * G + rank
        dgz.sample_uniform(g, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                           gen.batch_rng_seed(c.seed, j), bufs)
        torch.cuda.synchronize()
        n = int(bufs.sizes_host[-1])
        mbs.append((bufs.ids_sorted[:n].clone(), bufs.ids_sorted_pos[:n].clone(), n))
    rows = sum(m[2] for m in mbs)
    outd = torch.empty(max(m[2] for m in mbs) * R, dtype=torch.uint8, device="cuda")

    def timed(fn):
        for m in mbs[:2]:
            fn(*m)
        torch.cuda.synchronize()
        bar()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for m in mbs:
            fn(*m)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        t = torch.tensor([ms, rows * R], dtype=torch.float64, device="cpu" if same else "cuda")
        allv = [torch.zeros_like(t) for _ in range(G)]
        dist.all_gather(allv, t)
        return ms, [float(x[0]) for x in allv], sum(float(x[1]) for x in allv)

    res = {"alpha": alpha, "ranks": G, "same_device": same, "rows_per_rank": rows, "runs": []}
    ms, all_ms, tot = timed(lambda ids, pos, n: dgz.gather_perm(tb, ids, pos, outd, n=n))
    res["runs"].append({"cache": 0.0, "per_rank_gbs": [round(rows * R / m / 1e6, 2) for m in all_ms],
                        "aggregate_gbs": round(tot / max(all_ms) / 1e6, 2)})
    for frac in fracs:
        k = int(c.n_nodes * frac)
        cache = dgz.ShardedHotRowCache(tb, order[:k].contiguous())
        slots = torch.cat([cache.slot_map[m[0]] for m in mbs])
        hit = float((slots >= 0).float().mean())
        peer = float(((slots >= 0) & (slots % G != rank)).float().mean())
        ms, all_ms, tot = timed(lambda ids, pos, n: cache.gather(ids, outd, dst_pos=pos, n=n))
        res["runs"].append({"cache": frac, "cache_gb_total": round(k * R / 1e9, 2), "cache_gb_per_gpu": round(k * R / G / 1e9, 2),
                            "hit_rate_rank": round(hit, 4), "peer_hit_rate_rank": round(peer, 4),
                            "per_rank_gbs": [round(rows * R / m / 1e6, 2) for m in all_ms],
                            "aggregate_gbs": round(tot / max(all_ms) / 1e6, 2)})
        m = mbs[0]
        cache.gather(m[0], outd, dst_pos=m[1], n=m[2])
        ref = outd[:m[2] * R].clone()
        dgz.gather_perm(tb, m[0], m[1], outd, n=m[2])
        torch.cuda.synchronize()
        res["runs"][-1]["equal_to_uncached"] = bool(torch.equal(ref, outd[:m[2] * R]))
        cache.close()
        del cache
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(res), flush=True)
    tb.unregister()
    bar()
    buf.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
