"""Why a co-running consumer slows the gather on DISJOINT SMs: the sorted config-4 gather on a 16-SM
green-context partition, alone and beside co-runners on the other 132 SMs that stress different
shared resources -- pure ALU (dgz_probe_spin), an HBM-streaming copy (2 x 4 GiB buffers: DRAM
bandwidth), and an L2-resident copy (2 x 24 MiB: L2 bandwidth, little DRAM).  If only the DRAM
streamer hurts, the gather's GPU page walks (page-table reads from DRAM) are what it contends on.
    python tools/explore23_interference_hbm.py > gpurun_out/explore23_interference_hbm.jsonl"""
import json
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402

torch.cuda.set_device(0)
c = gen.CONFIGS[4]
L = len(c.fanouts)
buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
gen.fill_table(buf.ptr, c.table_bytes, c.seed)
table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
del off, col
sbs = []
for j in range(6):
    sb = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=False, local=False)
    dgz.sample_uniform(graph, torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda(), c.fanouts,
                       gen.batch_rng_seed(c.seed, j), sb)
    sbs.append(sb)
torch.cuda.synchronize()
nrows = sum(int(sb.sizes_host[-1]) for sb in sbs)
out = torch.empty(sbs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
big = [torch.empty(4 << 30, dtype=torch.uint8, device="cuda") for _ in range(2)]
small = [torch.empty(24 << 20, dtype=torch.uint8, device="cuda") for _ in range(2)]
sink = torch.zeros(4, dtype=torch.float32, device="cuda")

for k in (16, 148 - 16):
    part = dgz.Partition(k, -1, dgz.PARTITION_SPREAD)
    pcfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=8, flags=dgz.FLAG_DEEP)
    fs, cs = part.fetch_stream, part.compute_stream

    def corun(kind, stop):
        with torch.cuda.stream(cs):
            while not stop.is_set():
                for _ in range(8):
                    if kind == "hbm_copy":
                        big[1].copy_(big[0])
                    elif kind == "l2_copy":
                        for _ in range(40):
                            small[1].copy_(small[0])
                    elif kind == "alu_spin":
                        dgz.probe_spin(part.compute_sms * 4, 256, 200_000, sink, stream=cs)
                cs.synchronize()

    for kind in ("none", "alu_spin", "l2_copy", "hbm_copy", "none"):
        stop = threading.Event()
        th = None
        if kind != "none":
            th = threading.Thread(target=corun, args=(kind, stop))
            th.start()
            time.sleep(0.05)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(fs)
        for sb in sbs:
            dgz.gather_perm(table, sb.ids_sorted, sb.ids_sorted_pos, out, n=sb.bounds[-1], n_dev=sb.sizes_dev[L:L + 1],
                            cfg=pcfg, stream=fs)
        b.record(fs)
        b.synchronize()
        stop.set()
        if th:
            th.join()
        torch.cuda.synchronize()
        print(json.dumps({"gather_sms": part.fetch_sms, "corunner": kind, "corunner_sms": part.compute_sms,
                          "gather_gbs": round(nrows * c.row_bytes / a.elapsed_time(b) / 1e6, 2)}), flush=True)
    part.destroy()
table.unregister()
buf.free()
