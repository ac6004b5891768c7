"""Roofline of the stand-in consumer's kernels on a config-4-shaped last-hop block.

    python tools/consumer_roofline.py [--n-dst 172000] [--n-src 830000] [--dim 128] [--hidden 256] [--fanout 5]

Synthetic block (seeded): x [n_src, dim] fp32 in HBM (the gathered minibatch, larger than L2),
positions uniform over x, counts min(fanout, Poisson(14.4)) -- the last hop of config 4.  Times
dgz_aggregate_mean and dgz_sage_mean_linear with CUDA events (median of 20 launches after 5 warm-up),
and reports algorithmic HBM bytes per launch: x rows read (1 + cnt) x dim x 4 per dst row, cnt (4 B)
and the nbr block row (fanout x 4 B), y written (dim or hidden x 4 B), W (hidden x dim x 2 B, once)
-- and GEMM FLOPs 2 x n_dst x dim x hidden.  One JSON line per kernel.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_03330_b200 import dgz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-dst", type=int, default=172_000)
    ap.add_argument("--n-src", type=int, default=830_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--fanout", type=int, default=5)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    cnt = np.minimum(a.fanout, rng.poisson(14.4, size=a.n_dst)).astype(np.int32)
    loc = rng.integers(0, a.n_src, size=(a.n_dst, a.fanout)).astype(np.int32)
    x = torch.rand(a.n_src, a.dim, device="cuda")
    locd, cntd = torch.from_numpy(loc).cuda(), torch.from_numpy(cnt).cuda()
    w = (torch.randn(a.hidden, a.dim) / a.dim ** 0.5).to(torch.bfloat16).cuda()
    s = torch.cuda.Stream()
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
    except Exception:
        pass
    rows_read = float((1 + cnt.astype(np.int64)).sum()) * a.dim * 4
    idx = a.n_dst * (4 + a.fanout * 4)

    def run(name, launch, out_w, flops):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.iters)]
        with torch.cuda.stream(s):
            for _ in range(5):
                launch()
            for e0, e1 in ev:
                e0.record(s)
                launch()
                e1.record(s)
        torch.cuda.synchronize()
        ms = float(np.median([e0.elapsed_time(e1) for e0, e1 in ev]))
        byts = rows_read + idx + a.n_dst * out_w * 4 + (a.hidden * a.dim * 2 if flops else 0)
        line = {"kernel": name, "n_dst": a.n_dst, "n_src": a.n_src, "dim": a.dim, "fanout": a.fanout,
                "mean_cnt": round(float(cnt.mean()), 3), "ms": round(ms, 4), "alg_bytes": int(byts),
                "hbm_gbs": round(byts / ms / 1e6, 1)}
        if flops:
            line.update({"hidden": a.hidden, "gemm_tflops": round(flops / ms / 1e9, 2)})
        for k in ("hbm_copy_gbs", "hbm_gbs", "copy_gbs"):
            if k in peaks:
                line["hbm_peak_gbs"] = peaks[k]
                line["frac"] = round(line["hbm_gbs"] / peaks[k], 3)
                break
        print(json.dumps(line), flush=True)

    y1 = torch.empty(a.n_dst, a.dim, device="cuda")
    for cps in (0, 8):
        run(f"aggregate_mean ctas_per_sm={cps}",
            lambda: dgz.aggregate_mean(x.view(-1), a.dim, locd.view(-1), cntd, a.fanout, None, a.n_dst, y1, ctas_per_sm=cps,
                                       stream=s), a.dim, 0)
    y2 = torch.empty(a.n_dst, a.hidden, device="cuda")
    for cps in (0, 1, 2):
        run(f"sage_mean_linear ctas_per_sm={cps}",
            lambda: dgz.sage_mean_linear(x.view(-1), a.dim, locd.view(-1), cntd, a.fanout, None, a.n_dst, w, y2, ctas_per_sm=cps,
                                         stream=s), a.hidden, 2.0 * a.n_dst * a.dim * a.hidden)


if __name__ == "__main__":
    main()
