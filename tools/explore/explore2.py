"""Why do random-row zero-copy gathers stop near 25 GB/s?  Footprint / order / row-size / THP sweep."""
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


def out(**kw):
    print(json.dumps(kw), flush=True)


def ev_time(fn, iters=3, warm=1):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters


def meminfo(key):
    for line in open("/proc/meminfo"):
        if line.startswith(key):
            return line.strip()
    return None


def main():
    torch.cuda.set_device(0)
    total = 56_862_697_472
    mode = sys.argv[1] if len(sys.argv) > 1 else "thp"
    flags = dgz.HOST_HUGEPAGE if mode == "thp" else 0
    buf = dgz.HostBuffer(total + 4096, flags=flags)
    t = time.time()
    gen.fill_table(buf.ptr, total, 1)
    out(step="fill", s=time.time() - t, anon_huge=meminfo("AnonHugePages"), mode=mode)
    outd = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")

    # row-size sweep over the full footprint
    tables = {}
    for R in (128, 512, 2048, 4096):
        rows = total // R
        tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32) if R not in tables else tables[R]
        tables[R] = tb
        if R == 128:
            out(step="register", gpu_mem_delta=tb.info.gpu_mem_delta, register_s=tb.info.register_seconds)
        n = min(rows, (400 << 20) // R)
        ids = torch.from_numpy(gen.distinct_ids(rows, n, R)).cuda()
        for order in ("random", "sorted"):
            x = ids if order == "random" else torch.sort(ids).values
            tt = ev_time(lambda: dgz.gather(tb, x, outd, n=n))
            out(step="rowsize", R=R, order=order, n=n, gbs=n * R / tt / 1e9, mrows_s=n / tt / 1e6)
        tb.unregister()
        if R != 128:
            pass
    # footprint sweep at R = 512
    R = 512
    tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
    for gb in (0.0625, 0.25, 1, 4, 16, 56.8):
        rows = int(gb * 1e9) // R
        n = min(rows, 800_000)
        ids = torch.from_numpy(gen.distinct_ids(rows, n, 77)).cuda()
        tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n))
        out(step="footprint", gb=gb, n=n, gbs=n * R / tt / 1e9)
    # real sampler output order (config 4)
    c = gen.CONFIGS[4]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False)
    L = len(c.fanouts)
    res = []
    for j in range(6):
        seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda()
        dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, j), bufs)
        torch.cuda.synchronize()
        n = int(bufs.sizes_host[-1])
        tt = ev_time(lambda: dgz.gather(tb, bufs.ids, outd, n=n), iters=1, warm=0)
        res.append(n * R / tt / 1e9)
    out(step="sampler_order", gbs=res)
    # page-sharing: how many distinct 4K pages does a minibatch touch?
    ids = bufs.ids[:n].cpu().numpy()
    pages = np.unique((ids * R) >> 12).shape[0]
    pages2m = np.unique((ids * R) >> 21).shape[0]
    out(step="pages", rows=n, pages4k=int(pages), pages2m=int(pages2m))
    tb.unregister()
    buf.free()


if __name__ == "__main__":
    main()
