import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen, oracle
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
R, base, rows = 520, 8, 6000
buf = dgz.HostBuffer(rows * R + base + 4096)
arr = buf.numpy(); gen.fill_table(arr.ctypes.data + base, rows * R, 5)
host = arr[base:base + rows * R]
t = dgz.register_table(buf.ptr + base, rows, R // 4, dgz.F32)
idx = np.unique(np.concatenate([np.arange(10, 60), np.array([100, 101, 102, 777, 778])]))
want, _ = oracle.gather(host, R, idx)
ids = torch.from_numpy(idx).cuda(); pos = torch.arange(idx.shape[0], dtype=torch.int64, device="cuda")
out = torch.full((idx.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
for name, cfg in (("nomerge", dgz.gather_cfg(flags=1)), ("default", dgz.gather_cfg()),
                  ("u8_148x2", dgz.gather_cfg(sm_count=148, warps_per_cta=2)),
                  ("u16_148x2", dgz.gather_cfg(sm_count=148, warps_per_cta=2, flags=2)),
                  ("u8_1x1", dgz.gather_cfg(sm_count=1, warps_per_cta=1)),
                  ("u16_1x1", dgz.gather_cfg(sm_count=1, warps_per_cta=1, flags=2))):
    flags = name
    out.fill_(0xAB)
    dgz.gather_perm(t, ids, pos, out, cfg=cfg); torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(-1, R)
    bad = np.argwhere(got != want)
    print("flags", flags, "bad bytes", len(bad))
    rows_bad = sorted(set(bad[:, 0].tolist()))
    for r in rows_bad[:6]:
        bb = bad[bad[:, 0] == r][:, 1]
        print(" row", r, "id", idx[r], "a%128", (base + idx[r] * R) % 128, "bad byte range", bb.min(), bb.max(), len(bb),
              "got==0xAB", bool((got[r, bb] == 0xAB).all()))
# where did the wrong bytes come from?
out.fill_(0xAB)
dgz.gather_perm(t, ids, pos, out, cfg=dgz.gather_cfg()); torch.cuda.synchronize()
got = out.cpu().numpy().reshape(-1, R)
H = host.tobytes()
for r in (31, 50):
    wrong = bytes(got[r, :8])
    locs = []
    st = 0
    while True:
        k = H.find(wrong, st)
        if k < 0 or len(locs) > 3: break
        locs.append(k); st = k + 1
    print("row", r, "wrong bytes found at table offsets", locs, "-> row", [l // R for l in locs], "byte", [l % R for l in locs],
          "expected row", idx[r], "| row-1 id", idx[r-1])
