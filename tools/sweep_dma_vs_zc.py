"""Config 5 row-width sweep: the product zero-copy path vs the conventional CPU-gather + cudaMemcpy
baseline on the SAME random row lists.  256 MiB of uniformly random distinct rows per
width over the 56.9 GB buffer (base offset 0 and 4), useful GB/s (GB = 1e9).

  zc  : dgz_order_ids + dgz_gather_perm (address-sorted zero-copy gather, default launch)
  dma : torch.index_select with all host threads into pinned staging, 32 MiB chunks, each chunk's
        cudaMemcpyAsync H2D overlapping the CPU gather of the next (double-buffered)

    python tools/sweep_dma_vs_zc.py [--zc-only] [--widths=66,202,...] [--threads=T] > gpurun_out/sweep_dma_vs_zc.jsonl
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
threads = os.cpu_count() or 1
for a in sys.argv[1:]:
    if a.startswith("--threads="):         # e.g. the host-core share of one GPU on an 8-GPU box
        threads = int(a.split("=", 1)[1])
torch.set_num_threads(threads)
total = gen.CONFIGS[4].table_bytes
MANAGED = "--managed" in sys.argv   # zero-copy from a DGZ_HOST_MANAGED table; the CPU gather reads a THP copy
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_MANAGED if MANAGED else dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total + 4096, 9)
cpu_buf = buf
if MANAGED:
    cpu_buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table(cpu_buf.ptr, total + 4096, 9)
host_all = torch.from_numpy(cpu_buf.numpy(0, total + 4096))
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
CH = 32 << 20
stage = [torch.empty(CH + 4096, dtype=torch.uint8).pin_memory() for _ in range(2)]
cs = torch.cuda.Stream()
done = [torch.cuda.Event(), torch.cuda.Event()]


def dma_gather(host_rows, ids_cpu, R):
    n = ids_cpu.numel()
    per = max(1, CH // R)
    k = 0
    for c0 in range(0, n, per):
        p = k % 2
        done[p].synchronize()
        m = min(per, n - c0)
        st = stage[p][:m * R].view(m, R)
        torch.index_select(host_rows, 0, ids_cpu[c0:c0 + m], out=st)
        with torch.cuda.stream(cs):
            outd[c0 * R:(c0 + m) * R].view(m, R).copy_(st, non_blocking=True)
            done[p].record(cs)
        k += 1
    cs.synchronize()


WIDTHS = gen.SWEEP_ROW_BYTES
for a in sys.argv[1:]:
    if a.startswith("--widths="):          # e.g. --widths=66,202,1030 (fp16 rows with odd dims: 2 B aligned)
        WIDTHS = tuple(int(x) for x in a.split("=", 1)[1].split(","))
for R in WIDTHS:
    for base in (0, 4):
        rows = (total - base) // R
        n = min(rows, (256 << 20) // R)
        tb = dgz.register_table(buf.ptr + base, rows, R // 4 if R % 4 == 0 else R, dgz.F32 if R % 4 == 0 else dgz.U8)
        ids_np = gen.distinct_ids(rows, n, R * 7 + base)
        ids = torch.from_numpy(ids_np).cuda()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # zc: the product path, including the on-device address sort of the list
        for _ in range(2):
            srt, pos = dgz.order_ids(ids, rows)
            dgz.gather_perm(tb, srt, pos, outd, n=n)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            srt, pos = dgz.order_ids(ids, rows)
            dgz.gather_perm(tb, srt, pos, outd, n=n)
        b.record()
        torch.cuda.synchronize()
        t_zc = a.elapsed_time(b) / 3 * 1e-3
        rec = {"R": R, "base": base, "n": n, "table": "managed" if MANAGED else "registered",
               "zc_gbs": round(n * R / t_zc / 1e9, 2), "zc_mrows_s": round(n / t_zc / 1e6, 1)}
        if "--zc-only" not in sys.argv:
            # dma baseline on the same IDs
            host_rows = host_all[base:base + rows * R].view(rows, R)
            ids_cpu = torch.from_numpy(ids_np)
            dma_gather(host_rows, ids_cpu, R)
            t0 = time.perf_counter()
            for _ in range(2):
                dma_gather(host_rows, ids_cpu, R)
            t_dma = (time.perf_counter() - t0) / 2
            rec.update({"dma_gbs": round(n * R / t_dma / 1e9, 2), "zc_over_dma": round(t_dma / t_zc, 2), "dma_threads": threads})
        print(json.dumps(rec), flush=True)
        tb.unregister()
buf.free()
if cpu_buf is not buf:
    cpu_buf.free()
