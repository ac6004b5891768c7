"""Does a UVM mapping of host-resident memory escape the 64 KiB page-walk limit?

The same sorted gathers as tools/smallrow_study.py part B (256 MiB of random distinct rows per width
over 56.9 GB) and part A (fixed strides), from three host tables:
  reg     -- cudaHostRegister'd anonymous memory (the product's table, dgz_register_table);
  managed -- cudaMallocManaged, filled by the CPU, cudaMemAdviseSetPreferredLocation(CPU) +
             SetAccessedBy(GPU): pages stay in host memory, the GPU reads them through its mapping;
  hmm     -- (when the device reports pageableMemoryAccess) plain pageable memory read directly.
Same kernel, same launch (the host-table default plan).  Prints JSON lines.

    python tools/uvm_host_study.py [reg] [managed] [hmm] > gpurun_out/uvm_host_study.jsonl
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
kinds = [a for a in sys.argv[1:] if a in ("reg", "managed", "hmm")] or ["reg", "managed", "hmm"]
total = gen.CONFIGS[4].table_bytes
dev = torch.cuda.current_device()
err, pageable = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrPageableMemoryAccess, dev)
err2, ats = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrPageableMemoryAccessUsesHostPageTables, dev)
print(json.dumps({"pageable_memory_access": int(pageable), "uses_host_page_tables": int(ats)}), flush=True)
outd = torch.empty((256 << 20) + 4096, dtype=torch.uint8, device="cuda")
a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def table_of(kind):
    if kind == "reg":
        buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)
        gen.fill_table(buf.ptr, total, 9)
        return buf.ptr, buf.free, "registered"
    if kind == "managed":
        e, ptr = rt.cudaMallocManaged(total + 4096, rt.cudaMemAttachGlobal)
        assert e == rt.cudaError_t.cudaSuccess, e
        (e,) = rt.cudaMemAdvise(ptr, total + 4096, rt.cudaMemoryAdvise.cudaMemAdviseSetPreferredLocation, rt.cudaCpuDeviceId)
        assert e == rt.cudaError_t.cudaSuccess, e
        gen.fill_table(int(ptr), total, 9)          # CPU first touch: resident in host memory
        (e,) = rt.cudaMemAdvise(ptr, total + 4096, rt.cudaMemoryAdvise.cudaMemAdviseSetAccessedBy, dev)
        assert e == rt.cudaError_t.cudaSuccess, e
        return int(ptr), (lambda: rt.cudaFree(ptr)), "device"
    buf = dgz.HostBuffer(total + 4096, flags=dgz.HOST_HUGEPAGE)   # hmm: pageable, never registered
    gen.fill_table(buf.ptr, total, 9)
    return buf.ptr, buf.free, "device"


def timed(tb, ids, pos, n, cfg):
    a_ev.record()
    dgz.gather_perm(tb, ids, pos, outd, n=n, cfg=cfg)
    b_ev.record()
    torch.cuda.synchronize()
    return a_ev.elapsed_time(b_ev) * 1e-3


PLANS = {}
for kind in kinds:
    if kind == "hmm" and not pageable:
        print(json.dumps({"kind": "hmm", "skipped": "device reports no pageable memory access"}), flush=True)
        continue
    ptr, free, how = table_of(kind)
    for R in (64, 128, 256, 512, 1024):
        rows = total // R
        n = min(rows, (256 << 20) // R)
        if how == "registered":
            tb = dgz.register_table(ptr, rows, R // 4, dgz.F32)
        else:
            tb = dgz.DeviceTable(ptr, rows, R // 4, dgz.F32)
        # the launch the product uses for a host table of this shape (dgz_gather_plan of the registered
        # table, recorded by the "reg" pass; the measured shape rule otherwise)
        if how == "registered":
            plan = dgz.gather_plan(tb, n, True)
            PLANS[R] = plan
        plan = PLANS.get(R, {"sm_count": 148, "warps_per_cta": 2 if R >= 1024 else 1, "flags": dgz.FLAG_DEEP})
        cfg = dgz.gather_cfg(sm_count=plan["sm_count"], warps_per_cta=plan["warps_per_cta"], ctas_per_sm=1,
                             flags=plan["flags"])
        orderer = dgz.Orderer(n)
        ts = []
        for rep in range(3):
            ids = torch.from_numpy(gen.distinct_ids(rows, n, R * 31 + rep)).cuda()
            srt, pos = orderer.order(ids, rows)
            torch.cuda.synchronize()
            ts.append(timed(tb, srt, pos, n, cfg))
            if rep == 0:
                want = torch.from_numpy(np.ascontiguousarray(
                    np.ctypeslib.as_array((ctypes.c_uint8 * R).from_address(ptr + int(ids[7].item()) * R))))
                got = outd[7 * R:8 * R].cpu()
                ok = bool(torch.equal(got, want))
        t = float(np.median(ts[1:]))
        print(json.dumps({"kind": kind, "R": R, "n": n, "gbs": round(n * R / t / 1e9, 2), "mrows_s": round(n / t / 1e6, 1),
                          "first_ms": round(ts[0] * 1e3, 3), "ms": round(t * 1e3, 3), "row7_ok": ok,
                          "launch": [plan["sm_count"], plan["warps_per_cta"]]}), flush=True)
        tb.unregister()
    free()
