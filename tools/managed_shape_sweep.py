"""Launch shape of the sorted gather on a managed host table (DGZ_HOST_MANAGED, 2 MiB GPU pages): the
default plan was tuned on cudaHostRegister'd tables, where few rows in flight win because page walks
are the limit; without walks the link's request rate is.  256 MiB of fresh
sorted random distinct rows per point over the 56.9 GB table, median of 2 after a warm-up list.

    python tools/managed_shape_sweep.py > gpurun_out/managed_shape_sweep.jsonl
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
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_MANAGED)
gen.fill_table(buf.ptr, total, 9)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
SHAPES = [(148, 1, 1, 2), (148, 2, 1, 2), (148, 4, 1, 2), (148, 8, 1, 2), (148, 2, 2, 2), (148, 4, 2, 2),
          (148, 1, 1, 0), (148, 2, 1, 0), (74, 2, 1, 2), (74, 4, 1, 2)]   # (SMs, warps/CTA, CTAs/SM, flags)
for R in (64, 128, 256, 512, 2048):
    rows = total // R
    n = min(rows, (256 << 20) // R)
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    orderer = dgz.Orderer(n)
    default = dgz.gather_plan(tb, n, True)
    for shp in [None] + SHAPES:
        k, w, cps, fl = shp if shp is not None else (None, 0, 0, 0)
        cfg = None if k is None else dgz.gather_cfg(sm_count=k, warps_per_cta=w, ctas_per_sm=cps, flags=fl)
        ts = []
        for rep in range(3):
            ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 97 + rep + (0 if k is None else k * w * cps + fl))).cuda()
            srt, pos = orderer.order(ids, rows)
            torch.cuda.synchronize()
            a.record()
            dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
            b.record()
            torch.cuda.synchronize()
            if rep:
                ts.append(a.elapsed_time(b) * 1e-3)
        t = float(np.median(ts))
        shape = ("default " + json.dumps([default["sm_count"], default["warps_per_cta"], default["ctas"], default["flags"]])
                 if k is None else [k, w, cps, fl])
        print(json.dumps({"R": R, "shape": shape, "gbs": round(n * R / t / 1e9, 2), "mrows_s": round(n / t / 1e6, 1)}),
              flush=True)
    tb.unregister()
buf.free()
