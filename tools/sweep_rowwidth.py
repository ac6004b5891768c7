"""Config 5: row-width sweep (the fig:alignment_measurement analogue).

For each row width R (bytes) and table base offset, the config-4 host buffer (56.9 GB) is
reinterpreted as rows of R bytes; 256 MiB worth of distinct uniformly random row IDs, sorted by
address (as the sampler emits them), are gathered by every kernel variant:
  SEGMENT (product: per-row 128 B line plan), BULK (TMA), NAIVE (Listing 2 without the shift),
  SHIFT (Listing 2 with the circular shift).  GB/s = useful bytes / kernel time (CUDA events).
Also prints the request model's line-level efficiency per width (oracle/request_model.py is not
imported: the closed form L = ceil((o+R)/128), S = sectors is restated here for the report).

    python tools/sweep_rowwidth.py > profiles/r01/sweep_rowwidth.jsonl
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


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


def main():
    torch.cuda.set_device(0)
    total = gen.CONFIGS[4].table_bytes
    widths = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else list(gen.SWEEP_ROW_BYTES)
    bases = (0, 4)
    buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table(buf.ptr, total + 4096, 9)
    outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
    h = torch.from_numpy(buf.numpy(0, 256 << 20))
    t = ev_time(lambda: outd[:256 << 20].copy_(h, non_blocking=True))
    print(json.dumps({"dma_h2d_gbs": round((256 << 20) / t / 1e9, 2)}), flush=True)
    for R in widths:
        for base in bases:
            rows = (total - base) // R
            n = min(rows, (256 << 20) // R)
            tb = dgz.register_table(buf.ptr + base, rows, R // 4 if R % 4 == 0 else R, dgz.F32 if R % 4 == 0 else dgz.U8)
            ids = torch.sort(torch.from_numpy(gen.distinct_ids(rows, n, R * 7 + base)).cuda()).values
            rec = {"R": R, "base": base, "n": n}
            for name, var in (("segment", 1), ("bulk", 4), ("naive", 2), ("shift", 3)):
                cfg = dgz.gather_cfg(variant=var, flags=dgz.FLAG_DEEP if var == 1 else 0,
                                     warps_per_cta=2 if var == 1 else 0)
                try:
                    tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n, cfg=cfg))
                    rec[name] = round(n * R / tt / 1e9, 2)
                except Exception as e:  # e.g. BULK row limit
                    rec[name] = None
                    rec[name + "_err"] = str(e)[:80]
            o = [(base + i * R) % 128 for i in range(128)]
            lines = sum((x + R + 127) // 128 for x in o) / 128
            sectors = sum((x + R + 31) // 32 - x // 32 for x in o) / 128
            rec["lines_per_row"] = round(lines, 3)
            rec["payload_eff"] = round(R / (32 * sectors), 4)
            print(json.dumps(rec), flush=True)
            tb.unregister()
    buf.free()


if __name__ == "__main__":
    main()
