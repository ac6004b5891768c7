"""Exploration run on the B200 box: ceilings, gather variants, SM sweep, sampler timing.

    python tools/explore.py [--rows N] [--quick]

Prints JSON lines; not the bench (bench.py is).  Used to pick defaults and to write DESIGN.md.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


def ev_time(fn, iters=5, warm=2, stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(iters):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters


def out(**kw):
    print(json.dumps(kw), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=111_059_956)
    ap.add_argument("--R", type=int, default=512)
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    R, rows = a.R, a.rows
    nbytes = rows * R
    t0 = time.time()
    buf = dgz.HostBuffer(nbytes + 4096, flags=dgz.HOST_HUGEPAGE)
    t1 = time.time()
    gen.fill_table(buf.ptr, nbytes, 0x5EED + 4)
    t2 = time.time()
    table = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    t3 = time.time()
    info = table.info
    out(step="setup", table_gb=nbytes / 1e9, alloc_s=t1 - t0, fill_s=t2 - t1, register_s=t3 - t2,
        gpu_mem_delta=info.gpu_mem_delta, ratio=nbytes / max(info.gpu_mem_delta, 1), threads=os.cpu_count())

    # DMA ceiling
    h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    t = ev_time(lambda: d.copy_(h, non_blocking=True), iters=10)
    out(step="dma_h2d", gbs=(256 << 20) / t / 1e9)
    # DMA from the registered table itself (mapped region)
    hv = torch.from_numpy(buf.numpy(0, 256 << 20))
    t = ev_time(lambda: d.copy_(hv, non_blocking=True), iters=10)
    out(step="dma_h2d_registered", gbs=(256 << 20) / t / 1e9)
    del h

    sink = torch.zeros(2, dtype=torch.int64, device="cuda")
    probe_bytes = 2 << 30
    for sms in ([1, 2, 4, 8, 16, 148] if not a.quick else [4, 148]):
        for warps in (8, 32):
            for unroll in (4, 16):
                off = (sms * 7919 + warps * 31 + unroll) % 20 * (2 << 30)  # fresh region each config
                t = ev_time(lambda: dgz.probe_stream(info.dev_ptr + off, probe_bytes, sms, warps, unroll, sink),
                            iters=1, warm=0)
                out(step="zc_stream", sms=sms, warps=warps, unroll=unroll, gbs=probe_bytes / t / 1e9)

    # pointer chase RTT: chain through distinct 4 KiB-spaced lines of the table
    arr = buf.numpy(0, 64 << 20).view(np.int64)
    nsteps = 2000
    stride = 4096 // 8
    perm = np.random.default_rng(0).permutation(np.arange(1, nsteps + 1))
    cur = 0
    saved = arr[: (nsteps + 1) * stride: stride].copy()
    for p in perm:
        arr[cur * stride] = int(p) * stride
        cur = int(p)
    arr[cur * stride] = 0
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    dgz.probe_chase(info.dev_ptr, nsteps, cyc)
    torch.cuda.synchronize()
    c = cyc[0].item()
    clk = torch.cuda.clock_rate() if hasattr(torch.cuda, "clock_rate") else 1965
    out(step="rtt", cycles_per_hop=c / nsteps, us_at_max_clock=c / nsteps / 1965.0, clock_mhz_now=clk)
    arr[: (nsteps + 1) * stride: stride] = saved

    # gather variants on 937k distinct random rows (config-4-sized minibatch)
    n = 937_000
    outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
    idsets = [torch.from_numpy(gen.distinct_ids(rows, n, 1000 + i)).cuda() for i in range(4)]
    it = [0]

    def run(cfg):
        def f():
            dgz.gather(table, idsets[it[0] % 4], outd, n=n, cfg=cfg)
            it[0] += 1
        return f
    for variant in (dgz.GATHER_SEGMENT, dgz.GATHER_BULK, dgz.GATHER_NAIVE, dgz.GATHER_SHIFT):
        sms_list = [0] if variant in (dgz.GATHER_NAIVE, dgz.GATHER_SHIFT) else ([0, 1, 2, 4, 8, 16, 32, 74] if not a.quick else [0, 8])
        for sms in sms_list:
            for warps in ((0,) if variant in (2, 3) else (8, 16, 32)):
                cfg = dgz.gather_cfg(variant=variant, sm_count=sms, warps_per_cta=warps)
                t = ev_time(run(cfg), iters=4, warm=1)
                out(step="gather", variant=variant, sms=sms, warps=warps, ms=t * 1e3, gbs=n * R / t / 1e9)

    # sampler on the config-4 graph
    c = gen.CONFIGS[4]
    tg = time.time()
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    tg = time.time() - tg
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=True, local=True)
    seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(8)]
    k = [0]

    def samp():
        dgz.sample_uniform(g, seeds[k[0] % 8], c.fanouts, gen.batch_rng_seed(c.seed, k[0]), bufs)
        k[0] += 1
    t = ev_time(samp, iters=8, warm=2)
    out(step="sampler", gen_csr_s=tg, edges=int(off[-1]), ms=t * 1e3, sizes=bufs.sizes_host.tolist())
    table.unregister()
    buf.free()


if __name__ == "__main__":
    main()
