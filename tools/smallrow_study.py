"""Small-row sparse gather study: what bounds the address-sorted zero-copy gather of
rows < 512 B over the 56.9 GB pinned table?

Part A ("stride"): R-byte rows at a FIXED stride s through the table (sorted, one list per point, each
list on table pages no earlier list touched, so no translation is cached from before): rows/s as a
function of s separates the costs per row, per 4 KiB page, per 64 KiB (one 128 B line of 8 B PTEs) and
per 2 MiB region.
Part B ("random"): 256 MiB of uniformly random distinct rows per width (fresh list per repetition),
rows/s, and the distinct 4 KiB pages / 64 KiB regions / 2 MiB regions each list touches.

    python tools/smallrow_study.py [A] [B] > gpurun_out/smallrow_study.jsonl
    ncu ... python tools/smallrow_study.py B --ncu      (one launch per point, for the counters)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
NCU = "--ncu" in sys.argv
parts = [a for a in sys.argv[1:] if a in ("A", "B")] or ["A", "B"]
total = gen.CONFIGS[4].table_bytes
MANAGED = "--managed" in sys.argv    # the table in DGZ_HOST_MANAGED memory instead of cudaHostRegister'd
UNSORTED = "--unsorted" in sys.argv  # part B without the address sort
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_MANAGED if MANAGED else dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 9)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(tb, ids, pos, n, cfg=None, reps=1):
    a_ev.record()
    for _ in range(reps):
        dgz.gather_perm(tb, ids, pos, outd, n=n, cfg=cfg)
    b_ev.record()
    torch.cuda.synchronize()
    return a_ev.elapsed_time(b_ev) / reps * 1e-3


def distinct(x, shift):
    return int(np.unique(x >> shift).shape[0])


if "A" in parts:
    R = 128
    tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
    rows_total = total // R
    cursor = 0       # next unused table row: every list starts on fresh pages
    for s in (128, 1024, 4096, 8192, 16384, 32768, 65536, 131072, 262144, 1 << 20, 2 << 20, 8 << 20):
        step = s // R
        n = min(1 << 20, (rows_total - cursor) // step)
        if n < 1000:
            cursor = 0
            n = min(1 << 20, rows_total // step)
        for rep in range(2):
            if cursor + n * step > rows_total:
                cursor = 0
            ids = torch.arange(cursor, cursor + n * step, step, dtype=torch.int64, device="cuda")[:n]
            pos = torch.arange(n, dtype=torch.int64, device="cuda")
            cursor += n * step + (2 << 20) // R
            torch.cuda.synchronize()
            t = timed(tb, ids, pos, n)
            if rep == 0 and not NCU:
                continue      # first list warms the code path; report the second (fresh pages too)
            h = ids.cpu().numpy() * R
            rec = {"part": "A", "table": "managed" if MANAGED else "registered", "R": R, "stride": s, "n": n, "gbs": round(n * R / t / 1e9, 2), "mrows_s": round(n / t / 1e6, 1),
                   "pages4k": distinct(h, 12), "regions64k": distinct(h, 16), "regions2m": distinct(h, 21), "ms": round(t * 1e3, 3)}
            rec["m_pages4k_s"] = round(rec["pages4k"] / t / 1e6, 1)
            rec["m_regions64k_s"] = round(rec["regions64k"] / t / 1e6, 1)
            print(json.dumps(rec), flush=True)
            if NCU:
                break
    tb.unregister()

if "B" in parts:
    for R in (64, 128, 256, 512, 1024):
        rows = total // R
        n = min(rows, (256 << 20) // R)
        tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
        orderer = dgz.Orderer(n)
        res = []
        for rep in range(1 if NCU else 3):
            ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 31 + rep)).cuda()
            if UNSORTED:     # the list as drawn (no address order): positions are the identity
                srt, pos = ids, torch.arange(n, dtype=torch.int64, device="cuda")
            else:
                srt, pos = orderer.order(ids, rows)
            torch.cuda.synchronize()
            t = timed(tb, srt, pos, n)
            res.append(t)
            if rep == 0:
                h = srt.cpu().numpy() * R
                counts = {"pages4k": distinct(h, 12), "regions64k": distinct(h, 16), "regions2m": distinct(h, 21)}
        t = float(np.median(res))
        rec = {"part": "B", "table": "managed" if MANAGED else "registered", "sorted": not UNSORTED, "R": R, "n": n, "gbs": round(n * R / t / 1e9, 2), "mrows_s": round(n / t / 1e6, 1),
               "ms": round(t * 1e3, 3), **counts}
        rec["m_pages4k_s"] = round(counts["pages4k"] / t / 1e6, 1)
        rec["m_regions64k_s"] = round(counts["regions64k"] / t / 1e6, 1)
        print(json.dumps(rec), flush=True)
        tb.unregister()
buf.free()
