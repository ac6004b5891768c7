import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
R = int(sys.argv[1]); sms = int(sys.argv[2]); warps = int(sys.argv[3]); n = int(sys.argv[4])
total = 1 << 30
buf = dgz.HostBuffer(total, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, total, 5)
tb = dgz.register_table(buf.ptr, total // R, R // 4, dgz.F32)
outd = torch.empty(n * R, dtype=torch.uint8, device="cuda")
ids = torch.arange(n, dtype=torch.int64, device="cuda") % (total // R)
dgz.gather(tb, ids, outd, n=n, cfg=dgz.gather_cfg(variant=4, sm_count=sms, warps_per_cta=warps))
torch.cuda.synchronize()
import numpy as np
ok = np.array_equal(outd[:R * 8].cpu().numpy(), buf.numpy(0, R * 8))
print("ok", R, sms, warps, n, ok, flush=True)
