"""What stretches the consumer when the fetch runs beside it?  (overlap leg, DESIGN 5.1)

The a7 layer (dgz_sage_mean_linear, config-4 last-hop block, repeated to ~8.5 ms) runs on the whole GPU
on a plain stream while one co-runner occupies a green-context partition of k SMs (spread):
  none      -- the consumer alone
  spin      -- an ALU spin kernel, 1 CTA x W warps per partition SM (SM occupancy only, no memory)
  pcie      -- a zero-copy LDG.128 stream over a pinned host buffer (PCIe reads + L2, no HBM writes)
  gather    -- the product gather (sorted 512 B rows of a 16 GiB managed host table -> HBM)
Each co-runner is enqueued for longer than the consumer; the consumer's time (CUDA events on its
stream) is reported against its time alone.  JSON lines.

    python tools/explore/overlap_attrib.py [--sms 32] [--warps 2]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sms", type=int, default=32)
    ap.add_argument("--warps", type=int, default=2)
    ap.add_argument("--repeat", type=int, default=45)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(0)
    n_dst, n_src, dim, hidden, f = 172_000, 830_000, 128, 256, 5
    cnt = torch.from_numpy(np.minimum(f, rng.poisson(14.4, size=n_dst)).astype(np.int32)).cuda()
    loc = torch.from_numpy(rng.integers(0, n_src, size=(n_dst, f)).astype(np.int32)).cuda()
    x = torch.rand(n_src, dim, device="cuda")
    w = (torch.randn(hidden, dim) / dim ** 0.5).to(torch.bfloat16).cuda()
    y = torch.empty(n_dst, hidden, device="cuda")
    comp = torch.cuda.Stream()

    ym = torch.empty(n_dst, dim, device="cuda")
    mean_only = os.environ.get("ATTRIB_CONSUMER") == "mean"

    def consumer():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        if mean_only:
            dgz.aggregate_mean(x.view(-1), dim, loc.view(-1), cnt, f, None, n_dst, ym, repeat=a.repeat, stream=comp)
        else:
            dgz.sage_mean_linear(x.view(-1), dim, loc.view(-1), cnt, f, None, n_dst, w, y, repeat=a.repeat, stream=comp)
        e1.record(comp)
        return e0, e1

    # co-runner resources
    part = dgz.Partition(a.sms, -1, dgz.PARTITION_SPREAD)
    ps = part.fetch_stream
    sink = torch.zeros(1024, device="cuda")
    pin_bytes = 1 << 30
    pin = dgz.HostBuffer(pin_bytes, flags=dgz.HOST_HUGEPAGE)
    ptab = dgz.register_table(pin.ptr, pin_bytes // 128, 128, dgz.U8)
    rows, R = (16 << 30) // 512, 512
    tbuf = dgz.HostBuffer(rows * R + 4096, flags=dgz.HOST_MANAGED)
    gen.fill_table(tbuf.ptr, rows * R, 1)
    table = dgz.register_table(tbuf.ptr, rows, R // 4, dgz.F32)
    ids = torch.from_numpy(np.sort(gen.distinct_ids(rows, 828_000, 3))).cuda()
    out = torch.empty(828_000 * R, dtype=torch.uint8, device="cuda")
    gcfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=a.warps, flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)

    # round 2 also tried the BULK (TMA) gather with its ring capped at 24 KiB so it co-resides with the layer:
    # no better (24 SMs: 1.18x vs 1.10x stretch), so that flag was not kept
    bcfg = dgz.gather_cfg(variant=dgz.GATHER_BULK, sm_count=part.fetch_sms, warps_per_cta=4)
    prim = torch.cuda.Stream(priority=-1)   # primary context, high priority: a bounded grid, SMs chosen by the scheduler

    def corunner(kind, ms_target):
        """Enqueue ~ms_target of the co-runner on the partition stream (or, *_primary, a bounded grid of
        the same CTA count on a plain stream of the primary context)."""
        if kind == "spin_primary":
            dgz.probe_spin(part.fetch_sms, 32 * a.warps, int(ms_target * 1.9e6 / 4), sink, stream=prim)
        elif kind == "gather_primary":
            for _ in range(int(ms_target / 8) + 1):
                dgz.gather(table, ids, out, cfg=gcfg, stream=prim)
        elif kind in ("bulk", "bulk_primary"):   # TMA bulk copies into the shared-memory ring
            for _ in range(int(ms_target / 8) + 1):
                dgz.gather(table, ids, out, cfg=bcfg, stream=prim if kind == "bulk_primary" else ps)
        elif kind == "spin":
            dgz.probe_spin(part.fetch_sms, 32 * a.warps, int(ms_target * 1.9e6 / 4), sink, stream=ps)
        elif kind == "pcie":
            for _ in range(int(ms_target / 21) + 1):     # 1 GiB at ~50 GB/s ~ 21 ms
                dgz.probe_stream(ptab.info.dev_ptr, pin_bytes, part.fetch_sms, a.warps, 8, sink, stream=ps)
        elif kind == "gather":
            for _ in range(int(ms_target / 8) + 1):
                dgz.gather(table, ids, out, cfg=gcfg, stream=ps)

    def run(kind):
        torch.cuda.synchronize()
        if kind != "none":
            corunner(kind, 40.0)
        e0, e1 = consumer()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    for _ in range(2):
        run("none")
    base = float(np.median([run("none") for _ in range(3)]))
    dgz.gather(table, ids, out, cfg=gcfg, stream=ps)   # first touch of the managed table's GPU mapping
    for st, c_, what in ((ps, gcfg, "segment, partition"), (prim, gcfg, "segment, bounded grid"),
                         (ps, bcfg, "bulk small ring, partition"), (prim, bcfg, "bulk, bounded grid")):
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(st)
        for _ in range(4):
            dgz.gather(table, ids, out, cfg=c_, stream=st)
        g1.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"gather_alone_ms": round(g0.elapsed_time(g1) / 4, 3), "where": what}), flush=True)
    print(json.dumps({"corunner": "none", "consumer_ms": round(base, 3), "sms": part.fetch_sms, "warps": a.warps}), flush=True)
    kinds = os.environ.get("ATTRIB_KINDS", "spin,pcie,gather,spin_primary,gather_primary").split(",")
    for kind in kinds:
        t = float(np.median([run(kind) for _ in range(3)]))
        # the co-runner's own time beside the consumer (gathers only): 8 gathers back to back under the consumer
        g_ms = None
        if kind.startswith("gather") or kind.startswith("bulk"):
            st = prim if kind.endswith("primary") else ps
            c_ = bcfg if kind.startswith("bulk") else gcfg
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dgz.sage_mean_linear(x.view(-1), dim, loc.view(-1), cnt, f, None, n_dst, w, y, repeat=a.repeat * 8, stream=comp)
            g0.record(st)
            for _ in range(4):
                dgz.gather(table, ids, out, cfg=c_, stream=st)
            g1.record(st)
            torch.cuda.synchronize()
            g_ms = round(g0.elapsed_time(g1) / 4, 3)
        # the co-runner alone for the same wall time, to see whether it is slowed in turn
        print(json.dumps({"corunner": kind, "consumer_ms": round(t, 3), "stretch": round(t / base, 3),
                          "gather_ms_under_consumer": g_ms, "sms": part.fetch_sms, "warps": a.warps}), flush=True)
    torch.cuda.synchronize()
    table.unregister()
    ptab.unregister()
    part.destroy()


if __name__ == "__main__":
    main()
