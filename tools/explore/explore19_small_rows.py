"""Small rows (config 5, R = 64 / 128 / 256 B): launch-shape sweep of the sorted zero-copy gather
(warps per CTA x loads in flight x CTAs per SM x schedule) -- is the translation-bound rate set by
how many distinct pages are in flight?  256 MiB of sorted random distinct rows over the 56.9 GB buffer.
    python tools/explore19_small_rows.py > gpurun_out/explore19_small_rows.jsonl"""
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
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for R in (64, 128, 256):
    rows = total // R
    n = (256 << 20) // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    srt, pos = dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 13)).cuda(), rows)
    for sms, warps, cps, flags, sched in ((0, 0, 0, 0, 0), (148, 1, 1, 2, 0), (148, 2, 1, 2, 0), (148, 4, 1, 2, 0),
                                          (148, 8, 1, 2, 0), (148, 16, 1, 2, 0), (148, 16, 2, 2, 0), (148, 16, 4, 2, 0),
                                          (148, 2, 1, 0, 0), (148, 8, 1, 0, 0), (74, 4, 1, 2, 0), (37, 8, 1, 2, 0),
                                          (148, 2, 1, 2, 2), (148, 8, 1, 2, 2), (148, 16, 4, 2, 2)):
        cfg = dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, ctas_per_sm=cps, flags=flags, schedule=sched)
        dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(json.dumps({"R": R, "sms": sms, "warps": warps, "ctas_per_sm": cps, "deep": flags == 2, "blocked": sched == 2,
                          "gbs": round(n * R / ms / 1e6, 2), "mrows_s": round(n / ms / 1e3, 1)}), flush=True)
    tb.unregister()
buf.free()
