"""Sequential rows: is the zero-copy ceiling the same for LDG (SEGMENT) and TMA (BULK)?"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz

def out(**kw): print(json.dumps(kw), flush=True)
def ev_time(fn, iters=4, warm=1):
    for _ in range(warm): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / iters

torch.cuda.set_device(0)
total = 8 << 30
buf = dgz.HostBuffer(total, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 5)
outd = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for R in (512, 4096, 16384):
    tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
    n = (1 << 30) // R
    ids = torch.arange(n, dtype=torch.int64, device="cuda")
    for variant, sms, warps, flags in ((1, 148, 2, 2), (1, 148, 8, 2), (1, 8, 16, 2), (4, 148, 8, 0), (4, 32, 8, 0), (4, 8, 8, 0), (4, 148, 2, 0)):
        cfg = dgz.gather_cfg(variant=variant, sm_count=sms, warps_per_cta=warps, flags=flags)
        tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n, cfg=cfg))
        out(R=R, variant=variant, sms=sms, warps=warps, gbs=round(n * R / tt / 1e9, 2))
    tb.unregister()
# DMA reference on the same buffer
h = torch.from_numpy(buf.numpy(0, 1 << 30))
tt = ev_time(lambda: outd.copy_(h, non_blocking=True))
out(dma_gbs=round((1 << 30) / tt / 1e9, 2))
