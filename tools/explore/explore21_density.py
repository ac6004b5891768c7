"""Launch shape vs sample density for the sorted zero-copy gather: R x (bytes gathered) x (CTAs, warps),
all with 16 line loads per lane.  Density = gathered rows / table rows over the 56.9 GB buffer.
    python tools/explore21_density.py > gpurun_out/explore21_density.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
total = gen.CONFIGS[4].table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 9)
outd = torch.empty((1 << 30) + 4096, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
SHAPES = [(148, 1), (148, 2), (96, 1), (96, 2), (74, 1), (74, 2), (48, 2)]
for R in (128, 256, 512, 1024):
    rows = total // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    for mib in (32, 128, 512, 1024):
        n = (mib << 20) // R
        srt, pos = dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 19 + mib)).cuda(), rows)
        for sms, warps in SHAPES:
            cfg = dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, flags=dgz.FLAG_DEEP)
            dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
            torch.cuda.synchronize()
            reps = max(2, 512 // mib)
            a.record()
            for _ in range(reps):
                dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            print(json.dumps({"R": R, "mib": mib, "n": n, "gap_kb": round(total / n / 1024, 1), "sms": sms, "warps": warps,
                              "gbs": round(n * R / ms / 1e6, 2)}), flush=True)
        del srt, pos
    tb.unregister()
buf.free()
