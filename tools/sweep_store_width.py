"""Store-width check: rows whose width or base is only 2-byte aligned (fp16 rows of
odd dims) are stored with SW = 2 (eight u16 stores per 16 B line piece); 16 B-aligned rows with SW = 16.
Product path (dgz_order_ids + dgz_gather_perm, default launch), 256 MiB of fresh uniformly random
distinct rows per repetition over the 56.9 GB buffer, median of 3; the store width each point uses
is reported (SW = lowest set bit of R | base | 16).

    python tools/sweep_store_width.py > gpurun_out/sweep_store_width.jsonl
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
total = gen.CONFIGS[4].table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total + 4096, 9)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
POINTS = [  # (R bytes, dtype, base)
    (64, "f32", 0), (66, "f16", 0), (200, "f32", 0), (202, "f16", 0), (512, "f32", 0), (514, "f16", 0),
    (1024, "f32", 0), (1030, "f16", 0), (1032, "f32", 0), (1028, "f32", 0), (2048, "f32", 0), (2050, "f16", 0),
    (1024, "f16", 2), (1024, "f32", 4), (4096, "f32", 0), (4098, "f16", 0)]
for R, dt, base in POINTS:
    dtype = dgz.F16 if dt == "f16" else dgz.F32
    eb = dgz.ELEM_BYTES[dtype]
    rows = (total - base) // R
    n = min(rows, (256 << 20) // R)
    tb = dgz.register_table(buf.ptr + base, rows, R // eb, dtype)
    orderer = dgz.Orderer(n)
    ts = []
    for rep in range(4):
        ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 131 + base * 7 + rep)).cuda()
        srt, pos = orderer.order(ids, rows)
        torch.cuda.synchronize()
        a.record()
        dgz.gather_perm(tb, srt, pos, outd, n=n)
        b.record()
        torch.cuda.synchronize()
        if rep:
            ts.append(a.elapsed_time(b) * 1e-3)
    x = R | base | 16
    sw = x & -x
    t = float(np.median(ts))
    print(json.dumps({"R": R, "dtype": dt, "base": base, "sw": sw, "n": n, "gbs": round(n * R / t / 1e9, 2),
                      "mrows_s": round(n / t / 1e6, 1), "plan": dgz.gather_plan(tb, n, True)}), flush=True)
    tb.unregister()
buf.free()
