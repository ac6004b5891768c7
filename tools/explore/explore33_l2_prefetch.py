"""Can GPU-initiated zero-copy reads use larger PCIe requests?  The streaming probe over a 1 GiB pinned
buffer with the loads' L2 prefetch-size hint (.L2::64B/128B/256B) vs none, at several SM counts.
    python tools/explore33_l2_prefetch.py > gpurun_out/explore33_l2_prefetch.jsonl"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
nbytes = 1 << 30
buf = dgz.HostBuffer(nbytes, flags=dgz.HOST_HUGEPAGE)
buf.numpy()[::4096] = 1
t = dgz.register_table(buf.ptr, nbytes // 128, 128, dgz.U8)
sink = torch.zeros(2, dtype=torch.int64, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(2):
    for sms in (8, 32, 148):
        for pf in (0, 64, 128, 256):
            dgz.probe_stream_hint(t.info.dev_ptr, nbytes, sms, 32, pf, sink)
            torch.cuda.synchronize()
            a.record()
            for _ in range(4):
                dgz.probe_stream_hint(t.info.dev_ptr, nbytes, sms, 32, pf, sink)
            b.record()
            torch.cuda.synchronize()
            print(json.dumps({"rep": rep, "sms": sms, "l2_prefetch": pf,
                              "gbs": round(4 * nbytes / a.elapsed_time(b) / 1e6, 2)}), flush=True)
t.unregister()
buf.free()
