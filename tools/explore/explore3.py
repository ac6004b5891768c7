"""cudaHostRegister (4 KiB GPU pages) vs CUDA VMM host allocation: random-row gather rate."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz

def out(**kw): print(json.dumps(kw), flush=True)

def ev_time(fn, iters=3, warm=1):
    for _ in range(warm): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters

torch.cuda.set_device(0)
total = 56_862_697_472
f0 = torch.cuda.mem_get_info()[0]
t = time.time()
buf = dgz.HostBuffer(total, flags=dgz.HOST_VMM)
out(step="vmm_alloc", s=time.time() - t, gpu_mem_delta=f0 - torch.cuda.mem_get_info()[0], ptr=hex(buf.ptr))
t = time.time(); gen.fill_table(buf.ptr, total, 1); out(step="fill", s=time.time() - t)
outd = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
for R in (128, 512, 2048):
    rows = total // R
    tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    if R == 128: out(step="register", flags=tb.info.flags, delta=tb.info.gpu_mem_delta)
    n = min(rows, (400 << 20) // R)
    ids = torch.from_numpy(gen.distinct_ids(rows, n, R)).cuda()
    for order in ("random", "sorted"):
        x = ids if order == "random" else torch.sort(ids).values
        tt = ev_time(lambda: dgz.gather(tb, x, outd, n=n))
        out(step="rowsize", R=R, order=order, gbs=n * R / tt / 1e9, mrows_s=n / tt / 1e6)
    # correctness spot check
    got = outd[: 64 * R].cpu().numpy().reshape(64, R)
    hv = buf.numpy(0, rows * R).reshape(rows, R)
    xs = x[:64].cpu().numpy()
    assert np.array_equal(got, hv[xs]), "VMM gather mismatch"
    tb.unregister()
R = 512
tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
for gb in (1, 4, 16, 56.8):
    rows = int(gb * 1e9) // R; n = min(rows, 800_000)
    ids = torch.from_numpy(gen.distinct_ids(rows, n, 77)).cuda()
    for variant in (1, 4):
        tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n, cfg=dgz.gather_cfg(variant=variant)))
        out(step="footprint", gb=gb, variant=variant, gbs=n * R / tt / 1e9)
for sms in (1, 2, 4, 8, 16, 32):
    rows = total // R; n = 800_000
    ids = torch.from_numpy(gen.distinct_ids(rows, n, 5)).cuda()
    for variant in (1, 4):
        tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n, cfg=dgz.gather_cfg(variant=variant, sm_count=sms)))
        out(step="sm_sweep", sms=sms, variant=variant, gbs=n * R / tt / 1e9)
# DMA from VMM host memory
hv = torch.from_numpy(buf.numpy(0, 256 << 20))
d = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
tt = ev_time(lambda: d.copy_(hv, non_blocking=True), iters=5)
out(step="dma_from_vmm", gbs=(256 << 20) / tt / 1e9)
# export / import round trip in-process
fd = buf.export_fd()
b2 = dgz.HostBuffer(1 << 30, import_fd=fd)
out(step="import", same=bool(np.array_equal(b2.numpy(0, 4096), buf.numpy(0, 4096))), ptr2=hex(b2.ptr))
b2.free(); os.close(fd)
tb.unregister(); buf.free()
