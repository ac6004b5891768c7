"""The HBM ceiling for the a7 layer's access pattern: random 512 B row reads.

The layer reads, per destination row, its own row and ~5 random rows of the 425 MB gathered
minibatch (more than L2).  A sequential copy (MEASURED_PEAKS.json hbm_gbs) is not that pattern; this
measures what random row reads can reach on this GPU with the repo's own gather kernel on an
HBM-resident table (dgz_wrap_device_table, frontier = unsorted order, the All-in-GPU path):
  random   -- 1.03 M row IDs uniform over the 830 k-row table (the layer's neighbour reads)
  sorted   -- the same IDs in ascending order
Each: bytes read (n x R) and written (n x R) per launch / time (CUDA events, median of 10).

    python tools/explore/hbm_random_rows.py [--rows 830000] [--n 1032000] [--row-bytes 512]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2103_03330_b200 import dgz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=830_000)
    ap.add_argument("--n", type=int, default=1_032_000)
    ap.add_argument("--row-bytes", type=int, default=512)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    R = a.row_bytes
    tab = torch.randint(0, 255, (a.rows * R,), dtype=torch.uint8, device="cuda")
    t = dgz.DeviceTable(tab.data_ptr(), a.rows, R // 4, dgz.F32)
    rng = np.random.default_rng(1)
    ids = rng.integers(0, a.rows, size=a.n).astype(np.int64)
    out = torch.empty(a.n * R, dtype=torch.uint8, device="cuda")
    # read-only: the random-row read ceiling at several depths and warp counts (dgz_probe_rows)
    sink = torch.zeros(4, dtype=torch.int64, device="cuda")
    d = torch.from_numpy(ids).cuda()
    for warps in (8, 16, 32):
        for u in (1, 2, 4, 8, 16):
            for _ in range(2):
                dgz.probe_rows(tab.data_ptr(), R, d, 0, warps, u, sink)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                dgz.probe_rows(tab.data_ptr(), R, d, 0, warps, u, sink)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(json.dumps({"read_only": True, "warps_per_sm": warps, "rows_in_flight_per_warp": u, "n": a.n, "row_bytes": R,
                              "ms": round(ms, 4), "read_gbs": round(a.n * R / ms / 1e6, 1)}), flush=True)
    for name, idx in (("random", ids), ("sorted", np.sort(ids))):
        d = torch.from_numpy(idx).cuda()
        for _ in range(3):
            dgz.gather(t, d, out)
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dgz.gather(t, d, out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(json.dumps({"order": name, "rows": a.rows, "n": a.n, "row_bytes": R, "ms": round(ms, 4),
                          "read_gbs": round(a.n * R / ms / 1e6, 1), "read_plus_write_gbs": round(2 * a.n * R / ms / 1e6, 1)}),
              flush=True)


if __name__ == "__main__":
    main()
