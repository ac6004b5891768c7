"""compute-sanitizer target (test infrastructure: checks against the oracle): every gather variant
(SEGMENT, NAIVE, SHIFT, BULK) and the sorted gather at three row widths (tools/sanitize.sh)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen, oracle
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
for R, base in ((512, 0), (2408, 8), (100, 4)):
    rows = 3000
    buf = dgz.HostBuffer(rows * R + 8192)
    gen.fill_table(buf.ptr + base, rows * R, R)
    t = dgz.register_table(buf.ptr + base, rows, R // 4, dgz.F32)
    idx = gen.random_ids(rows, 2000, 1)
    want, _ = oracle.gather(buf.numpy(base, rows * R), R, idx)
    out = torch.empty(2000 * R, dtype=torch.uint8, device="cuda")
    ids = torch.from_numpy(idx).cuda()
    for v in (1, 2, 3, 4):
        dgz.gather(t, ids, out, cfg=dgz.gather_cfg(variant=v, sm_count=4))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), (R, v)
    o = np.argsort(idx, kind="stable")
    for cfg in (None, dgz.gather_cfg(sm_count=6, warps_per_cta=3, flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)):
        dgz.gather_perm(t, torch.from_numpy(idx[o]).cuda(), torch.from_numpy(o.astype(np.int64)).cuda(), out, cfg=cfg)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    # the hot-row cache (two local shards) and the work-counter schedule through it
    cache = dgz.HotRowCache(t, torch.from_numpy(idx[:300].copy()).cuda(), 2)
    for cfg in (None, dgz.gather_cfg(flags=dgz.FLAG_DYNAMIC)):
        cache.gather(torch.from_numpy(idx[o]).cuda(), out, dst_pos=torch.from_numpy(o.astype(np.int64)).cuda(), cfg=cfg)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    del cache
    t.unregister(); buf.free()
# BULK with more consumer warps than ring slots (40 KiB rows, default warps)
R, rows = 40960, 64
buf = dgz.HostBuffer(rows * R + 8192)
gen.fill_table(buf.ptr, rows * R, 3)
t = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
idx = gen.random_ids(rows, 150, 2)
want, _ = oracle.gather(buf.numpy(0, rows * R), R, idx)
out = torch.empty(150 * R, dtype=torch.uint8, device="cuda")
dgz.gather(t, torch.from_numpy(idx).cuda(), out, cfg=dgz.gather_cfg(variant=dgz.GATHER_BULK, sm_count=2))
torch.cuda.synchronize()
assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
t.unregister(); buf.free()
# the stand-in consumer
x = torch.from_numpy(gen.float_table(2000 * 64, 1)).cuda()
loc = torch.from_numpy(gen.random_ids(2000, 500 * 5, 4).astype(np.int32)).cuda()
cnt = torch.full((500,), 5, dtype=torch.int32, device="cuda")
y = torch.empty(500 * 64, dtype=torch.float32, device="cuda")
dgz.aggregate_mean(x, 64, loc, cnt, 5, None, 500, y, repeat=2)
torch.cuda.synchronize()
# the a7 layer (tcgen05 MMA + TMEM): K 64 (direct epilogue) and K 128 (epilogue staged through shared memory)
for d in (64, 128, 320):   # 320: K in three chunks
    xs = torch.from_numpy(gen.float_table(2000 * d, 2)).cuda()
    w = (torch.randn(256, d) / d ** 0.5).to(torch.bfloat16).cuda()
    ys = torch.empty(500 * 256, dtype=torch.float32, device="cuda")
    dgz.sage_mean_linear(xs, d, loc, cnt, 5, None, 500, w, ys, repeat=2)
    dgz.sage_mean_linear(xs, d, loc, cnt, 5, None, 500, w, ys, ctas_per_sm=1, sm_count=2)
    torch.cuda.synchronize()
    assert torch.isfinite(ys).all()
print("bulk/segment/naive/shift/dynamic/cached/aggregate/sage ok")
