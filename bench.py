#!/usr/bin/env python
"""Benchmark of the hot path of arXiv 2103.03330 on B200: GPU sampling + zero-copy feature gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 4]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one process per GPU)

A step = one minibatch fetch: seeds of global batch j (j = i*G + rank)
-> dgz_sample_uniform (3-hop uniform sampling on the GPU, CSR in HBM) -> dgz_gather_perm
(rows of the pinned, mapped host table read by zero-copy over PCIe into HBM).  Metric:
gathered feature GB/s (useful bytes n*R / time, GB = 1e9), whole-job aggregate over ranks.
Inputs are resident (CSR and per-step seeds in HBM, table pinned) before the timed region;
the 56.9 GB table and fresh minibatches every step are far larger than the 126 MB L2.

Rank 0 prints ONE JSON line.  ``--impl reference`` times the CPU oracle (oracle/, a plain
single-threaded C sampler + row gather) on the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import dgz_inputs as gen  # noqa: E402

METRIC = "gathered feature GB/s per GPU and aggregate at 1/2/4/8 B200 vs PCIe Gen5 roofline"
UNIT = "GB/s"


# ----------------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------------
class Dist:
    def __init__(self, want_gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.same_device = os.environ.get("DGZ_BENCH_SAME_DEVICE") == "1"  # N ranks on one GPU (test only)
        if self.same_device:
            self.local = 0
        if self.world > 1:
            import torch.distributed as dist
            backend = "nccl" if (torch.cuda.is_available() and not self.same_device) else "gloo"
            self.backend = backend
            if torch.cuda.is_available():
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.pg = dist
        elif torch.cuda.is_available():
            torch.cuda.set_device(0)
        if want_gpus != self.world and self.rank == 0:
            print(f"# note: --gpus {want_gpus} but WORLD_SIZE {self.world}; using {self.world}", file=sys.stderr)

    def barrier(self):
        if self.pg:
            if self.backend == "nccl":
                self.pg.barrier(device_ids=[self.local])
            else:
                self.pg.barrier()

    def allreduce(self, vals, op="sum"):
        if not self.pg:
            return list(vals)
        dev = "cuda" if self.backend == "nccl" else "cpu"
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM if op == "sum" else self.pg.ReduceOp.MAX)
        return t.cpu().tolist()

    def bcast_obj(self, obj):
        if not self.pg:
            return obj
        lst = [obj]
        self.pg.broadcast_object_list(lst, src=0)
        return lst[0]

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((float(r[3]) for r in self.rows if len(r) > 8 and r[3].replace(".", "").isdigit()),
                                   default=None)}


# ----------------------------------------------------------------------------------------------
# shared inputs
# ----------------------------------------------------------------------------------------------
def make_table(cfg, d: Dist, dgz):
    """Host feature table: one copy on the box, registered by every rank."""
    nbytes = cfg.table_bytes
    if d.world == 1:
        buf = dgz.HostBuffer(nbytes + 4096, flags=dgz.HOST_HUGEPAGE)
        t0 = time.time()
        gen.fill_table(buf.ptr, nbytes, cfg.seed)
        fill_s = time.time() - t0
    else:
        name = f"/dgz_bench_c{cfg.cid}_{os.environ.get('MASTER_PORT', '0')}"
        fill_s = 0.0
        if d.rank == 0:   # interleaved over the sockets' memory when the box has several NUMA nodes
            buf = dgz.HostBuffer(nbytes + 4096, shm_name=name, create=True,
                                 flags=dgz.HOST_HUGEPAGE | dgz.HOST_NUMA_INTERLEAVE)
            t0 = time.time()
            gen.set_threads(os.cpu_count() or 1)      # the other ranks are waiting: use every core
            gen.fill_table(buf.ptr, nbytes, cfg.seed)
            gen.set_threads(max(1, (os.cpu_count() or 1) // d.world))
            fill_s = time.time() - t0
        d.barrier()
        if d.rank != 0:
            buf = dgz.HostBuffer(nbytes + 4096, shm_name=name, create=False, flags=dgz.HOST_HUGEPAGE)
        d.barrier()
        if d.rank == 0:
            buf.unlink()   # the mappings stay valid; the name does not outlive the run
    return buf, fill_s


def make_csr(cfg, d: Dist, dgz):
    """The graph's CSR on the host: plain arrays for N = 1; for N > 1 rank 0 generates it once
    into shared /dev/shm mappings that every rank maps (one host copy per box, not one per rank).
    Returns (offsets int64 view, cols int32 view, n_edges, keep-alive buffers)."""
    if d.world == 1:
        off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed)
        return off, col, int(off[-1]), []
    base = f"/dgz_bench_csr{cfg.cid}_{os.environ.get('MASTER_PORT', '0')}"
    bufs = []
    e = None
    if d.rank == 0:
        def alloc(nb):
            b = dgz.HostBuffer(nb + 4096, shm_name=f"{base}_{len(bufs)}", create=True, flags=dgz.HOST_NUMA_INTERLEAVE)
            bufs.append(b)
            return b.ptr
        gen.set_threads(os.cpu_count() or 1)
        _, _, e = gen.gen_csr_into(cfg.n_nodes, cfg.avg_degree, cfg.seed, alloc)
        gen.set_threads(max(1, (os.cpu_count() or 1) // d.world))
    e = int(d.bcast_obj(e))
    if d.rank != 0:
        for i, nb in enumerate(((cfg.n_nodes + 1) * 8, max(e * 4, 1))):
            bufs.append(dgz.HostBuffer(nb + 4096, shm_name=f"{base}_{i}", create=False))
    d.barrier()
    if d.rank == 0:
        for b in bufs:
            b.unlink()
    off = bufs[0].numpy(0, (cfg.n_nodes + 1) * 8).view(np.int64)
    col = bufs[1].numpy(0, e * 4).view(np.int32)
    return off, col, e, bufs


def ev():
    return torch.cuda.Event(enable_timing=True)


def measure_ceilings(dgz, d: Dist):
    """In-run PCIe ceilings, every rank at once after a barrier (the per-link figure is this
    rank's; the aggregate = sum of bytes / max time over ranks is the host/root-complex limit
    the N-GPU value is compared with): H2D DMA from pinned memory, zero-copy streaming read."""
    h = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    h[::4096] = 1                                   # touch every page of the staging buffer
    dbuf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(40):                             # warm-up: the first ~50 copies ramp from ~43 to ~55 GB/s
        dbuf.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    trials, agg = [], []
    for _ in range(8):  # best of 8 x (10 copies of 256 MiB), all ranks concurrently
        torch.cuda.synchronize()
        d.barrier()
        a.record()
        for _ in range(10):
            dbuf.copy_(h, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        el = a.elapsed_time(b) * 1e-3
        trials.append(10 * (256 << 20) / el / 1e9)
        tot, mx = d.allreduce([10.0 * (256 << 20)], "sum")[0], d.allreduce([el], "max")[0]
        agg.append(tot / mx / 1e9)
    dma = max(trials)
    del h
    sink = torch.zeros(2, dtype=torch.int64, device="cuda")
    zbytes = 1 << 30
    pbuf = dgz.HostBuffer(zbytes, flags=dgz.HOST_HUGEPAGE)
    pbuf.numpy()[::4096] = 1
    ptab = dgz.register_table(pbuf.ptr, zbytes // 128, 128, dgz.U8)
    dgz.probe_stream(ptab.info.dev_ptr, zbytes, 8, 32, 8, sink)
    torch.cuda.synchronize()
    d.barrier()
    a.record()
    for _ in range(4):
        dgz.probe_stream(ptab.info.dev_ptr, zbytes, 8, 32, 8, sink)
    b.record()
    torch.cuda.synchronize()
    el = a.elapsed_time(b) * 1e-3
    zc = 4 * zbytes / el / 1e9
    zc_agg = d.allreduce([4.0 * zbytes], "sum")[0] / d.allreduce([el], "max")[0] / 1e9
    ptab.unregister()
    pbuf.free()
    del dbuf
    return {"h2d_dma_gbs": round(dma, 2), "h2d_dma_trials": [round(x, 2) for x in trials], "zc_stream_gbs": round(zc, 2),
            "ranks": d.world, "h2d_dma_aggregate_gbs": round(max(agg), 2), "zc_stream_aggregate_gbs": round(zc_agg, 2),
            "how": "every rank at once after a barrier: best of 8 x (cudaMemcpyAsync 256 MiB pinned H2D x10) after 40 "
                   "warm-up copies; zero-copy "
                   "LDG.128 stream over a 1 GiB pinned buffer x4 on 8 SMs; aggregate = sum bytes / max time over ranks"}


def hbm_peak() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling
    guide's fallback 6650 GB/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def load_profile_traffic(cid):
    """(dram bytes per gather launch, summary) from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "r01", "ncu_gather_summary.json")
    try:
        with open(p) as f:
            c = json.load(f).get(f"config{cid}")
        if not c:
            return None, None
        return int(c["dram_bytes_per_launch"]), {k: v for k, v in c.items() if k != "launches"}
    except Exception:
        return None, None


# ----------------------------------------------------------------------------------------------
# our implementation
# ----------------------------------------------------------------------------------------------
def run_ours(args, d: Dist):
    from paper_2103_03330_b200 import dgz
    from paper_2103_03330_b200.pipeline import MinibatchFetcher, calibrated_fetcher

    cfg = gen.CONFIGS[args.config]
    R = cfg.row_bytes
    L = len(cfg.fanouts)
    t_setup = time.time()
    gen.set_threads(max(1, (os.cpu_count() or 1) // d.world))
    buf, fill_s = make_table(cfg, d, dgz)
    table = dgz.register_table(buf.ptr, cfg.n_nodes, cfg.dim, dgz.F32)
    info = table.info
    t0 = time.time()
    off, col, n_edges, csr_bufs = make_csr(cfg, d, dgz)
    csr_s = time.time() - t0
    if args.csr == "host":    # zero-copy CSR (NEXT-3): the sampler reads the host arrays over PCIe
        graph = dgz.HostGraph(off.ctypes.data, col.ctypes.data, cfg.n_nodes, n_edges, False)
    else:                     # CSR replicated in each GPU's HBM
        graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())

    K, W = args.steps, args.warmup
    G, rank = d.world, d.rank
    batches = [i * G + rank for i in range(W + K)]
    seeds_host = [torch.from_numpy(gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j)) for j in batches]
    seeds_dev = [x.cuda() for x in seeds_host]
    rng = [gen.batch_rng_seed(cfg.seed, j) for j in batches]

    gflags = dgz.FLAG_DYNAMIC if args.dynamic else 0
    gcfg = (dgz.gather_cfg(sm_count=args.gather_sms, warps_per_cta=args.gather_warps, flags=gflags)
            if (args.gather_sms or args.gather_warps or gflags) else None)
    sm_count_all = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    choice = None
    if args.sampler_sms is None and not args.graphs and args.csr == "hbm":
        # the pipeline's shape is picked by measurement on the warm-up minibatches, before the timed
        # region (pipeline.calibrated_fetcher)
        fetcher, choice = calibrated_fetcher(table, graph, cfg.fanouts, cfg.batch, seeds_dev[:W], rng[:W], slots=2,
                                             gather_cfg=gcfg, blocks=True)
    else:
        fetcher = MinibatchFetcher(table, graph, cfg.fanouts, cfg.batch, slots=2, gather_cfg=gcfg, blocks=True,
                                   sampler_sms=args.sampler_sms, graphs=args.graphs)
    cap = fetcher.bufs[0].bounds[-1]
    n_steps = torch.zeros(W + K, dtype=torch.int64, device="cuda")
    ceilings = measure_ceilings(dgz, d)
    mbs = []

    def step(i):
        mbs.append(fetcher.fetch(seeds_dev[i], rng[i], timing=True, count_into=n_steps[i:i + 1]))

    for i in range(W):
        step(i)
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    launches0 = dgz.kernel_launches()
    replays0 = fetcher.graph_replays
    t_start, t_end = ev(), ev()
    with ClockSampler(d.local) as clk:
        t_start.record(fetcher.sample_stream)
        for i in range(W, W + K):
            step(i)
        fetcher.stream.wait_stream(fetcher.sample_stream)
        t_end.record(fetcher.stream)
        torch.cuda.synchronize()
    # kernels launched by libdgz calls, plus those replayed inside CUDA graphs (--graphs)
    launches = dgz.kernel_launches() - launches0 + (fetcher.graph_replays - replays0) * fetcher.graph_kernels
    d.barrier()
    torch.cuda.synchronize()
    dgz.check_errors(table)
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    ns = n_steps.cpu().tolist()[W:]
    bytes_rank = float(sum(ns) * R)
    tm = [mbs[i].timing for i in range(W, W + K)]
    gather_ms = [t[1].elapsed_time(t[2]) for t in tm]
    step_ms = [t[0].elapsed_time(t[2]) for t in tm]
    tot_bytes, = d.allreduce([bytes_rank], "sum")
    max_el, = d.allreduce([elapsed], "max")
    value = tot_bytes / max_el / 1e9
    per_gpu = bytes_rank / elapsed / 1e9
    gather_gbs = float(np.mean(ns)) * R / (float(np.mean(gather_ms)) * 1e-3) / 1e9

    # keep the last two minibatches for the oracle parity check (cpu_baseline leg)
    last = {}
    for i in (W + K - 2, W + K - 1):
        p = i % 2
        n = ns[i - W]
        last[batches[i]] = (mbs[i].bufs.ids[:n].cpu().numpy(), mbs[i].rows[:n].cpu().numpy(), rng[i],
                            seeds_host[i].numpy())

    # ---- end-to-end through the public API: pinned host seeds -> H2D -> sample -> gather -> D2H |U|
    e2e = run_e2e(fetcher, cfg, seeds_host, rng, W, K, d)

    # ---- minibatch-fetch latency, unpipelined: sampling then gather of one minibatch on one stream
    lat = run_latency(fetcher, cfg, seeds_dev, rng, min(K, 16))

    # ---- overlap with a stand-in consumer (steps a5-a7)
    overlap = (run_overlap(dgz, fetcher, cfg, seeds_dev, rng, W, K, args.overlap_warps)
               if (args.overlap and rank == 0) else None)

    # ---- baselines (rank 0 only, N=1 at most the box's cores): oracle + CPU-gather+memcpy
    cpu_base = dma_base = parity = None
    if not args.no_baselines:
        dma_base = run_dma_baseline(cfg, buf, fetcher, graph, seeds_dev, rng, W, K, d)   # every rank, concurrently
        if rank == 0:   # parity of the last two minibatches always; the oracle's timing at N = 1 only
            cpu_base, parity = run_oracle_leg(cfg, buf.ptr, off, col, last, d, budget=20.0 if G == 1 else 0.0)

    clocks = clk.summary()
    sm_count = torch.cuda.get_device_properties(0).multi_processor_count
    traffic, traffic_detail = load_profile_traffic(cfg.cid)
    peak = ceilings["h2d_dma_gbs"]
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": G, "steps": K, "warmup": W,
        "ms_per_step": round(max_el / K * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 (fp32 rows moved as bytes)", "data": "synthetic",
        "config": {"workload": f"config{cfg.cid} {cfg.name}: {cfg.n_nodes} nodes, {n_edges} edges "
                               f"(Poisson avg deg {cfg.avg_degree}), {cfg.dim}x fp32 = {R} B rows, "
                               f"{cfg.table_bytes / 1e9:.1f} GB pinned host table, fanouts {list(cfg.fanouts)}, "
                               f"{cfg.batch} seeds per GPU per step",
                   "global_batch": cfg.batch * G, "parallelism": f"dp{G} (seed partition j mod G)",
                   "l2": "inputs larger than L2 (56.9 GB table, fresh minibatch every step)",
                   "pipeline": fetcher.mode, "pipeline_choice": choice,
                   "csr": "HBM (replicated per GPU)" if args.csr == "hbm" else "pinned host memory, sampled by zero-copy",
                   "gather": dict(dgz.gather_plan(table, cap, True, gcfg),
                                  order="address-sorted + inverse permutation (dgz_gather_perm)")},
        "per_gpu_gbs": round(per_gpu, 3),
        "roofline": {"bound": "pcie", "achieved": round(gather_gbs, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(gather_gbs / peak, 4), "traffic": traffic, "traffic_detail": traffic_detail,
                     "kernel": "gather_segment_kernel (dgz_gather_perm)",
                     "peak_source": "measured in this run: cudaMemcpyAsync H2D from pinned memory (PCIe Gen5 x16); "
                                    "MEASURED_PEAKS.json has no PCIe figure",
                     "algorithmic_bytes_per_launch": round(float(np.mean(ns)) * R),
                     "gather_ms_mean": round(float(np.mean(gather_ms)), 4),
                     "zc_stream_frac": round(gather_gbs / ceilings["zc_stream_gbs"], 4),
                     "hbm_write_frac": round(gather_gbs / hbm_peak(), 5),
                     "aggregate": {"achieved": round(value, 3), "peak": ceilings["h2d_dma_aggregate_gbs"],
                                   "frac": round(value / ceilings["h2d_dma_aggregate_gbs"], 4),
                                   "zc_peak": ceilings["zc_stream_aggregate_gbs"],
                                   "what": f"whole-job step GB/s over {G} rank(s) vs the H2D DMA / zero-copy ceilings "
                                           "measured on all ranks at once (host root-complex limit)"}},
        "ceilings": ceilings,
        "latency_ms": {"fetch": lat,
                       "pipelined": {"gather_p10": pct(gather_ms, 10), "gather_p50": pct(gather_ms, 50),
                                     "gather_p90": pct(gather_ms, 90), "sample_to_gather_end_p50": pct(step_ms, 50),
                                     "note": "in the pipeline the sampling of j+1 starts during the gather of j, so "
                                             "sample start -> gather end spans about two gathers"}},
        "rows_per_step_mean": round(float(np.mean(ns)), 1),
        "cpu_baseline": cpu_base, "dma_baseline": dma_base, "parity": parity,
        "e2e": e2e, "overlap": overlap,
        "gpu_launches": int(launches), "gpu_launches_per_step": round(launches / K, 2),
        "clocks": clocks,
        "setup": {"table_fill_s": round(fill_s, 2), "register_s": round(info.register_seconds, 2),
                  "gpu_mem_mapping_bytes": info.gpu_mem_delta,
                  "mapping_ratio": round(cfg.table_bytes / max(info.gpu_mem_delta, 1), 1),
                  "csr_gen_s": round(csr_s, 2), "total_s": round(time.time() - t_setup, 1), "sms": sm_count,
                  "host_numa_nodes": dgz.host_numa_nodes(),
                  "host_table_policy": "anonymous THP mapping (first touch)" if G == 1 else
                                       "/dev/shm object shared by the ranks, NUMA-interleaved"},
    }
    fetcher.close()
    if args.csr == "host":
        graph.close()
    table.unregister()
    buf.free()
    for b in csr_bufs:
        b.free()
    return line


def pct(xs, q):
    return round(float(np.percentile(xs, q)), 4)


def run_latency(fetcher, cfg, seeds_dev, rng, n):
    """Minibatch-fetch latency without pipelining: on one stream, sample (whole GPU) then gather,
    events around each phase; p10/p50/p90 over n fresh minibatches."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    f = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, sampler_sms=0)
    for i in range(2):
        f.fetch(seeds_dev[i], rng[i]).event.synchronize()
    samp, gath, tot = [], [], []
    for i in range(n):
        mb = f.fetch(seeds_dev[i], rng[i], timing=True)
        mb.event.synchronize()
        t0, t1, t2 = mb.timing
        samp.append(t0.elapsed_time(t1))
        gath.append(t1.elapsed_time(t2))
        tot.append(t0.elapsed_time(t2))
    out = {}
    for k, xs in (("sample", samp), ("gather", gath), ("sample_plus_gather", tot)):
        out.update({f"{k}_p10": pct(xs, 10), f"{k}_p50": pct(xs, 50), f"{k}_p90": pct(xs, 90)})
    out["minibatches"] = n
    return out


def run_e2e(fetcher, cfg, seeds_host, rng, W, K, d: Dist):
    """Same metric through the public API with host-resident inputs: every step the seeds go H2D
    from pinned memory inside fetch(), and the step's result (|U|, a D2H copy) is read on the
    host -- one step behind, as a double-buffered user loop would, so the host read of step j-1
    overlaps the fetch of step j."""
    R = cfg.row_bytes
    pinned = [x.pin_memory() for x in seeds_host]

    def loop(lo, hi):
        total, prev = 0, None
        for i in range(lo, hi):
            mb = fetcher.fetch(pinned[i], rng[i])
            if prev is not None:
                total += prev.sizes()[-1]
            prev = mb
        return total + prev.sizes()[-1]
    loop(0, W)
    torch.cuda.synchronize()
    d.barrier()
    t0 = time.perf_counter()
    total = loop(W, W + K)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    tot, = d.allreduce([float(total * R)], "sum")
    mx, = d.allreduce([el], "max")
    L = len(cfg.fanouts)
    return {"value": round(tot / mx / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": cfg.batch * 8,
            "d2h_bytes_per_step": (L + 1) * 8, "ms_per_step": round(mx / K * 1e3, 4),
            "how": "MinibatchFetcher.fetch(pinned host seeds) each step + host read of each step's |U| (one step "
                   "behind), wall clock"}


def run_overlap(dgz, fetcher, cfg, seeds_dev, rng, W, K, overlap_warps=0):
    """Exposed fetch time with a stand-in GraphSAGE mean-aggregation consumer (a5-a7) and the
    SM-partition sweep (a6; the B200 analogue of the paper's MPS ratio sweep, fig:mps_bandwidth):
    the fetch runs on a green-context partition of k SMs (dgz_partition, spread over the GPCs),
    the consumer on the other 148 - k, and step j+1 is fetched while step j is consumed."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    dim = cfg.dim
    L = len(cfg.fanouts)
    nstep = min(K, 8)
    ev2 = (ev(), ev())

    def consume(comp, mb, repeat, y, nb, cb):
        dgz.aggregate_mean(mb.rows.view(torch.float32).view(-1), dim, mb.bufs.local[nb:], mb.bufs.cnt[cb:], cfg.fanouts[L - 1],
                           mb.bufs.sizes_dev[L - 1:L], mb.bufs.bounds[L - 1], y, repeat=repeat, stream=comp)

    def measure(f, comp, repeat=None, t_target=None):
        y = torch.empty((f.bufs[0].bounds[L - 1], dim), dtype=torch.float32, device="cuda")
        nb = sum(f.bufs[0].bounds[k] * cfg.fanouts[k] for k in range(L - 1))
        cb = sum(f.bufs[0].bounds[k] for k in range(L - 1))
        a, b = ev2
        for i in range(2):
            f.fetch(seeds_dev[i], rng[i])
        torch.cuda.synchronize()
        a.record(f.stream)
        for i in range(nstep):
            f.fetch(seeds_dev[i], rng[i])
        b.record(f.stream)
        torch.cuda.synchronize()
        t_g = a.elapsed_time(b) / nstep
        mb = f.fetch(seeds_dev[0], rng[0])
        mb.event.synchronize()

        def cons_alone(rep):
            torch.cuda.synchronize()
            a.record(comp)
            for _ in range(nstep):
                consume(comp, mb, rep, y, nb, cb)
            b.record(comp)
            torch.cuda.synchronize()
            return a.elapsed_time(b) / nstep
        if repeat is None:
            repeat = 8
            for _ in range(3):
                repeat = max(1, int(round(repeat * (t_target or t_g) / cons_alone(repeat))))
        t_c = cons_alone(repeat)
        torch.cuda.synchronize()
        mbs = [f.fetch(seeds_dev[0], rng[0])]
        a.record(comp)
        for i in range(1, nstep + 1):
            nxt = f.fetch(seeds_dev[i % len(rng)], rng[i % len(rng)])
            cur = mbs[-1]
            comp.wait_event(cur.event)
            consume(comp, cur, repeat, y, nb, cb)
            f.release(cur, comp)
            mbs.append(nxt)
        comp.wait_event(mbs[-1].event)
        b.record(comp)
        torch.cuda.synchronize()
        t_o = a.elapsed_time(b) / nstep
        return t_g, t_c, t_o, repeat

    f0 = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, sampler_sms=0)
    comp0 = torch.cuda.Stream()
    t_g0, t_c0, t_o0, repeat = measure(f0, comp0)
    del f0
    rows = [{"partition": "none (whole GPU, high-priority fetch stream)", "fetch_sms": 148, "t_fetch_ms": round(t_g0, 3),
             "t_consumer_ms": round(t_c0, 3), "t_step_overlapped_ms": round(t_o0, 3),
             "exposed_fetch_ms": round(max(0.0, t_o0 - t_c0), 3)}]
    # partition shapes: k SMs spread over every GPC, or k contiguous SMs of the split (DESIGN 5:
    # the gather's rate depends strongly and reproducibly on WHICH SMs it gets, explore25)
    for k, pflags in ((8, dgz.PARTITION_SPREAD), (16, dgz.PARTITION_SPREAD), (24, dgz.PARTITION_SPREAD),
                      (32, dgz.PARTITION_SPREAD), (16, 0), (24, 0)):
        try:
            part = dgz.Partition(k, -1, pflags)
        except Exception as e:  # green contexts unavailable: report and skip
            rows.append({"fetch_sms": k, "error": str(e)[:200]})
            continue
        shape = "spread over the GPCs" if pflags else "contiguous"
        # grid sized to the partition: one 8-warp CTA per SM, 16 line loads per lane (explore15)
        # work-counter batches (a partition's slower SMs take fewer batches, explore28) and few warps
        # per SM: beside a DRAM-heavy consumer the page walks slow down and fewer rows in flight win
        w = overlap_warps or max(2, 64 // part.fetch_sms)   # ~64 warps in all (8 SMs x 8 ... 32 SMs x 2)
        pcfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=w, flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)
        # sampler placement: in front of the gather on the small partition, or in the consumer's stream
        # between consumer steps (its full-partition bitmap passes then run beside the gather and slow
        # its page walks, but it leaves the small partition; DESIGN 5) -- both measured
        for where in ("fetch partition", "consumer stream"):
            f = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, fetch_stream=part.fetch_stream,
                                 gather_cfg=pcfg, sample_stream=part.compute_stream if where == "consumer stream" else None)
            t_g, t_c, t_o, _ = measure(f, part.compute_stream, repeat=repeat)
            rows.append({"partition": f"green context ({shape}), sampler in the {where}", "fetch_sms": part.fetch_sms,
                         "warps_per_sm": w,
                         "compute_sms": part.compute_sms,
                         "t_fetch_ms": round(t_g, 3), "t_consumer_ms": round(t_c, 3), "t_step_overlapped_ms": round(t_o, 3),
                         "exposed_fetch_ms": round(max(0.0, t_o - t_c), 3),
                         "fetch_gbs_alone": round(float(f.bufs[0].sizes_host[-1]) * cfg.row_bytes / t_g / 1e6, 2)})
        del f
        torch.cuda.synchronize()
        part.destroy()
    best = min((r for r in rows if "t_step_overlapped_ms" in r), key=lambda r: r["t_step_overlapped_ms"])
    return {"t_fetch_ms": round(t_g0, 3), "consumer_repeat": repeat, "serial_ms": round(t_g0 + t_c0, 3), "best": best,
            "hidden_frac_best": round(1 - best["exposed_fetch_ms"] / t_g0, 3), "sweep": rows,
            "consumer": "dgz_aggregate_mean over the last hop's block, non-persistent launches, repeated to T_c ~ T_fetch",
            "partition_gather": (f"{overlap_warps} warps per SM" if overlap_warps else "max(2, 64 / SMs) warps per SM")
                                + ", 16 loads per lane, work-counter batches"}


def run_oracle_leg(cfg, table_addr, off, col, last, d: Dist, budget: float = 20.0):
    """cpu_baseline: the oracle as it stands (single-threaded C) on a bounded sample of the
    same workload (about `budget` seconds; none when 0: N > 1), plus a full-size exact parity
    check of the GPU's last two minibatches."""
    import oracle
    R = cfg.row_bytes
    parity = {"batches": [], "exact": True}
    t_total, bytes_total, nb = 0.0, 0, 0
    for j, (U_gpu, rows_gpu, rs, seeds) in last.items():
        t0 = time.perf_counter()
        s, outb = oracle.sample_and_gather(off, col, seeds, cfg.fanouts, rs, table_addr, cfg.n_nodes, R)
        t_total += time.perf_counter() - t0
        n = s.U.shape[0]
        bytes_total += n * R
        nb += 1
        ok_u = bool(np.array_equal(s.U, U_gpu))
        ok_rows = ok_u and bool(np.array_equal(outb[:n * R].reshape(n, R), rows_gpu))
        parity["batches"].append({"j": int(j), "rows": int(n), "ids_equal": ok_u, "rows_equal": ok_rows})
        parity["exact"] &= ok_u and ok_rows
    # more minibatches (not compared) until ~budget seconds of oracle work
    j = 10_000_000
    while t_total < budget and nb < 40:
        seeds = gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j)
        rs = gen.batch_rng_seed(cfg.seed, j)
        t0 = time.perf_counter()
        s, _ = oracle.sample_and_gather(off, col, seeds, cfg.fanouts, rs, table_addr, cfg.n_nodes, R)
        t_total += time.perf_counter() - t0
        bytes_total += s.U.shape[0] * R
        nb += 1
        j += 1
    if budget <= 0:
        return None, parity
    return ({"value": round(bytes_total / t_total / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
             "sample": f"{nb} config{cfg.cid} minibatches (sample + gather, {t_total:.1f} s single-threaded C)",
             "s_per_minibatch": round(t_total / nb, 3), "host_cores": os.cpu_count()}, parity)


def run_dma_baseline(cfg, buf, fetcher, graph, seeds_dev, rng, W, K, d: Dist):
    """The paper's DMA-based method: CPU gathers the sampled rows into a pinned
    staging buffer with T threads, then cudaMemcpyAsync H2D; double-buffered so the CPU gather
    of j+1 overlaps the copy of j.  Same IDs as the GPU path (sampled on the GPU beforehand)."""
    R = cfg.row_bytes
    threads = max(1, (os.cpu_count() or 1) // d.world)
    torch.set_num_threads(threads)
    nb = min(K, 8)
    ids = []
    for i in range(nb):
        mb = fetcher.fetch(seeds_dev[i], rng[i])
        n = mb.sizes()[-1]
        ids.append(torch.from_numpy(mb.bufs.ids[:n].cpu().numpy()))
    host = torch.from_numpy(buf.numpy(0, cfg.table_bytes)).view(cfg.n_nodes, R)
    cap = max(x.numel() for x in ids)
    stage = [torch.empty((cap, R), dtype=torch.uint8).pin_memory() for _ in range(2)]
    dst = torch.empty((cap, R), dtype=torch.uint8, device="cuda")
    cs = torch.cuda.Stream()
    done = [torch.cuda.Event(), torch.cuda.Event()]
    torch.index_select(host, 0, ids[0], out=stage[0][:ids[0].numel()])  # warm
    torch.cuda.synchronize()
    d.barrier()
    t0 = time.perf_counter()
    total = 0
    for i in range(nb):
        p = i % 2
        done[p].synchronize()
        n = ids[i].numel()
        torch.index_select(host, 0, ids[i], out=stage[p][:n])
        with torch.cuda.stream(cs):
            dst[:n].copy_(stage[p][:n], non_blocking=True)
            done[p].record(cs)
        total += n * R
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    tot, = d.allreduce([float(total)], "sum")
    mx, = d.allreduce([el], "max")
    return {"value": round(tot / mx / 1e9, 3), "unit": UNIT, "threads_per_rank": threads, "ranks": d.world,
            "minibatches_per_rank": nb, "per_gpu_gbs": round(total / el / 1e9, 3),
            "how": "paper's DMA-based method (P:650-651): torch.index_select into pinned staging (host cores / G threads "
                   "per rank) + cudaMemcpyAsync, double-buffered, all ranks concurrently; aggregate = sum bytes / max time"}


# ----------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ----------------------------------------------------------------------------------------------
def run_reference(args, d: Dist):
    import oracle
    if d.rank != 0:
        return None
    cfg = gen.CONFIGS[args.config]
    R = cfg.row_bytes
    nbytes = cfg.table_bytes
    raw = np.empty(nbytes + 64, dtype=np.uint8)
    gen.fill_table(raw, nbytes, cfg.seed)
    off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed)
    out = np.empty(sum(gen.sample_bound(cfg.n_nodes, cfg.batch, cfg.fanouts)[-1:]) * R, dtype=np.uint8)
    K, W = args.steps, args.warmup

    def one(j):
        seeds = gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j)
        s, _ = oracle.sample_and_gather(off, col, seeds, cfg.fanouts, gen.batch_rng_seed(cfg.seed, j), raw.ctypes.data,
                                        cfg.n_nodes, R, out=out)
        return s.U.shape[0]
    for i in range(W):
        one(i)
    t0 = time.perf_counter()
    tot = 0
    for i in range(W, W + K):
        tot += one(i)
    el = time.perf_counter() - t0
    value = tot * R / el / 1e9
    return {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": d.world,
            "steps": K, "warmup": W, "ms_per_step": round(el / K * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8 (fp32 rows moved as bytes)", "data": "synthetic",
            "config": {"workload": f"config{cfg.cid} {cfg.name}", "global_batch": cfg.batch, "parallelism": "cpu (rank 0 only)"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{K} config{cfg.cid} minibatches, one per step (sample + gather, single-threaded C)"},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4])
    ap.add_argument("--gather-sms", type=int, default=0)
    ap.add_argument("--gather-warps", type=int, default=0)
    ap.add_argument("--sampler-sms", type=int, default=None,
                    help="SMs of the green-context sampler partition (0 = sample and gather back to back; "
                         "default 8 with the CSR in HBM, 0 with --csr host)")
    ap.add_argument("--graphs", action="store_true", help="replay sampler + gather as one CUDA graph per slot")
    ap.add_argument("--csr", default="hbm", choices=["hbm", "host"],
                    help="CSR replicated in HBM (default) or left in pinned host memory and sampled by zero-copy")
    ap.add_argument("--dynamic", action="store_true", help="gather batches from a work counter (DGZ_GATHER_FLAG_DYNAMIC)")
    ap.add_argument("--overlap-warps", type=int, default=0,
                    help="warps per SM of the overlap sweep's partition gathers (0: ~64 warps in all, at least 2 per SM)")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false")
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"
    d = Dist(args.gpus)
    try:
        line = run_reference(args, d) if args.impl == "reference" else run_ours(args, d)
        if d.rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    finally:
        d.close()


if __name__ == "__main__":
    main()
