"""Small rows (translation-bound) on different SM sets: 256 MiB of sorted random rows of R = 128 /
256 / 512 B gathered on the whole GPU (default launch) and on green-context partitions of explicit
SM-group sets (windows, strides, halves), 1 and 2 warps per SM, fresh lists for every point.
    python tools/explore27_small_rows_sm_sets.py > gpurun_out/explore27.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
ng, per = dgz.partition_groups()
total = gen.CONFIGS[4].table_bytes
buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 9)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
seed = [0]
SETS = {"whole GPU": None, "groups 0-36 (half)": list(range(0, 37)), "groups 37-73 (half)": list(range(37, 74)),
        "every 2nd group": list(range(0, ng, 2)), "groups 8-31 (24 groups)": list(range(8, 32)),
        "groups 16-23": list(range(16, 24)), "every 3rd group": list(range(0, ng, 3))}
for R in (128, 256, 512):
    rows = total // R
    n = (256 << 20) // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    for name, groups in SETS.items():
        for w in ((None,) if groups is None else (1, 2)):
            seed[0] += 1
            srt, pos = dgz.order_ids(torch.from_numpy(gen.distinct_ids(rows, n, R * 1000 + seed[0])).cuda(), rows)
            part = None
            if groups is None:
                s, cfg = torch.cuda.current_stream(), None
            else:
                part = dgz.Partition(0, -1, groups=groups)
                s, cfg = part.fetch_stream, dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=w, flags=dgz.FLAG_DEEP)
            dgz.gather_perm(tb, srt[:4096], pos[:4096], outd, n=4096, cfg=cfg, stream=s)   # warm-up: module load, flag
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            dgz.gather_perm(tb, srt, pos, outd, n=n, cfg=cfg, stream=s)
            b.record(s)
            torch.cuda.synchronize()
            print(json.dumps({"R": R, "set": name, "sms": part.fetch_sms if part else 148, "warps": w,
                              "gbs": round(n * R / a.elapsed_time(b) / 1e6, 2)}), flush=True)
            if part:
                part.destroy()
    tb.unregister()
buf.free()
