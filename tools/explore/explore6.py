"""Can the GPU map the host table with large pages?  cudaHostAlloc / hugetlbfs / THP / VMM."""
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
mode = sys.argv[1]
total = 56_862_697_472
R = 512; rows = total // R
flags = {"thp": dgz.HOST_HUGEPAGE, "cudapin": dgz.HOST_CUDA_PINNED, "huge2m": dgz.HOST_HUGETLB_2M, "huge1g": dgz.HOST_HUGETLB_1G}[mode]
if mode == "huge2m":
    open("/proc/sys/vm/nr_hugepages", "w").write(str(total // (2 << 20) + 64))
    out(nr_hugepages=open("/proc/sys/vm/nr_hugepages").read().strip())
if mode == "huge1g":
    p = "/sys/kernel/mm/hugepages/hugepages-1048576kB/nr_hugepages"
    try:
        open(p, "w").write(str(total // (1 << 30) + 2)); out(nr_1g=open(p).read().strip())
    except Exception as e:
        out(err=repr(e))
f0 = torch.cuda.mem_get_info()[0]
t = time.time()
buf = dgz.HostBuffer(total + (2 << 20), flags=flags)
out(step="alloc", mode=mode, s=round(time.time() - t, 2), gpu_delta_alloc=f0 - torch.cuda.mem_get_info()[0])
t = time.time(); gen.fill_table(buf.ptr, total, 1); out(step="fill", s=round(time.time() - t, 2))
f1 = torch.cuda.mem_get_info()[0]
t = time.time()
tb = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
out(step="register", s=round(time.time() - t, 2), gpu_delta_reg=f1 - torch.cuda.mem_get_info()[0], info_delta=tb.info.gpu_mem_delta)
n = 800_000
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
ids = torch.from_numpy(gen.distinct_ids(rows, n, 3)).cuda()
tt = ev_time(lambda: dgz.gather(tb, ids, outd, n=n))
out(step="random", gbs=n * R / tt / 1e9)
srt, order = torch.sort(ids)
tt = ev_time(lambda: dgz.gather_perm(tb, srt, order, outd, n=n))
out(step="sorted_perm", gbs=n * R / tt / 1e9)
got = outd[:R * 16].cpu().numpy().reshape(16, R)
hv = buf.numpy(0, total).reshape(rows, R)
out(step="check", ok=bool(np.array_equal(got, hv[ids[:16].cpu().numpy()])))
tb.unregister(); buf.free()
