"""torchrun worker for tests/test_gpu_cache_ipc.py: every rank (all on cuda:0, gloo) maps the
same /dev/shm table, owns one shard of a ShardedHotRowCache and reads the other ranks' shards
through CUDA IPC; its cached gathers must equal the oracle's byte for byte."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import dgz_inputs as gen  # noqa: E402
import oracle  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    R, rows, base = int(os.environ.get("CACHE_R", "400")), 50_000, int(os.environ.get("CACHE_BASE", "0"))
    name = f"/dgz_cache_ipc_{os.environ['MASTER_PORT']}"
    nbytes = rows * R + base + 4096
    if rank == 0:
        buf = dgz.HostBuffer(nbytes, shm_name=name, create=True)
        gen.fill_table(buf.ptr + base, rows * R, 77)
    dist.barrier()
    if rank != 0:
        buf = dgz.HostBuffer(nbytes, shm_name=name, create=False)
    dist.barrier()
    if rank == 0:
        buf.unlink()
    table = dgz.register_table(buf.ptr + base, rows, R // 4, dgz.F32)
    host = buf.numpy(base, rows * R)
    hot = torch.from_numpy(gen.distinct_ids(rows, 12_000, 1)).cuda()
    cache = dgz.ShardedHotRowCache(table, hot)
    assert cache.G == G and all(cache.view.shards[g] for g in range(G))
    for trial in range(3):
        idx_np = gen.random_ids(rows, 30_000, seed=100 * rank + trial)
        want, bad = oracle.gather(host, R, idx_np)
        assert bad == 0
        idx = torch.from_numpy(idx_np).cuda()
        out = torch.full((idx_np.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        cache.gather(idx, out)                                     # unsorted, identity positions
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), f"rank {rank} unsorted"
        srt, pos = dgz.order_ids(idx, rows)
        out.fill_(0xAB)
        cache.gather(srt, out, dst_pos=pos)                        # address-sorted, scattered back
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), f"rank {rank} sorted"
    hits = int(np.isin(idx_np, hot.cpu().numpy()).sum())
    dgz.check_errors(table)
    cache.close()
    table.unregister()
    buf.free()
    print(f"rank {rank}/{G} ok: {hits} of {idx_np.shape[0]} rows served from {G} HBM shards", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
