cat > /tmp/san_bulk2.py <<'PY'
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import dgz_inputs as gen
from paper_2103_03330_b200 import dgz
torch.cuda.set_device(0)
R=512; rows=3000
buf = dgz.HostBuffer(rows * R + 8192)
gen.fill_table(buf.ptr, rows * R, R)
t = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
idx = torch.from_numpy(gen.random_ids(rows, 2000, 1)).cuda()
out = torch.empty(2000 * R, dtype=torch.uint8, device="cuda")
dgz.gather(t, idx, out, cfg=dgz.gather_cfg(variant=4, sm_count=2))
torch.cuda.synchronize()
print("done")
PY
timeout 600 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 6 python /tmp/san_bulk2.py 2>&1 | head -60
