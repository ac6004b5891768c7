"""ncu evidence for the request plan (SURVEY 8(a) a4', 8(c) "pins"): sysmem sectors and L2 requests
that the gather kernels actually issue, per launch, for row widths that exercise the alignment
logic.  Run under ncu; `tests/test_sector_evidence.py` compares the committed counts with the
oracle's request model on the same regenerated IDs.

    ncu --metrics <see profiles/r01/README.md> --csv --log-file gpurun_out/sector_evidence.csv \
        python tools/sector_evidence.py gpurun_out/sector_evidence_manifest.json
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

N = 2048
WIDTHS = (100, 400, 480, 512, 516, 1028, 2408)
BASES = (0, 4)
VARIANTS = (("segment", dgz.GATHER_SEGMENT), ("naive", dgz.GATHER_NAIVE), ("shift", dgz.GATHER_SHIFT))
TABLE_BYTES = 2_000_000_000


def main(manifest_path):
    torch.cuda.set_device(0)
    buf = dgz.HostBuffer(TABLE_BYTES + 8192)
    gen.fill_table(buf.ptr, TABLE_BYTES + 4096, 5)
    out = torch.empty(N * max(WIDTHS) + 64, dtype=torch.uint8, device="cuda")
    launches = []
    for R in WIDTHS:
        for base in BASES:
            rows = TABLE_BYTES // R
            t = dgz.register_table(buf.ptr + base, rows, R // 4, dgz.F32)
            seed = R * 100 + base
            ids_np = gen.distinct_ids(rows, N, seed)
            ids = torch.from_numpy(ids_np).cuda()
            for name, v in VARIANTS:
                dgz.gather(t, ids, out, cfg=dgz.gather_cfg(variant=v))
                launches.append({"R": R, "base": base, "n": N, "rows": rows, "seed": seed, "variant": name})
            order = np.argsort(ids_np, kind="stable")
            srt = torch.from_numpy(ids_np[order]).cuda()
            pos = torch.from_numpy(order.astype(np.int64)).cuda()
            dgz.gather_perm(t, srt, pos, out, n=N)
            launches.append({"R": R, "base": base, "n": N, "rows": rows, "seed": seed, "variant": "segment_sorted_merge"})
            torch.cuda.synchronize()
            t.unregister()
    buf.free()
    with open(manifest_path, "w") as f:
        json.dump(launches, f, indent=0)


if __name__ == "__main__":
    main(sys.argv[1])
