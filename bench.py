#!/usr/bin/env python
"""Benchmark of the hot path of arXiv 2103.03330 on B200: GPU sampling + zero-copy feature gather.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1..5]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one process per GPU)

Configs 1-4 (BASELINE.json configs[0..3]): a step = one minibatch fetch:
seeds of global batch j (j = i*G + rank) -> dgz_sample_uniform (layered uniform sampling on the
GPU, CSR in HBM) -> dgz_gather_perm (rows of the pinned, mapped host table read by zero-copy over
PCIe into HBM).  ``--cache-frac f`` adds the HBM hot-row cache sharded over the ranks (NEXT-1) on
the power-law variant of the graph.

Config 5 (configs[4], the row-width sweep): ``--config 5 --row-bytes R --base B --dtype f32|f16``;
a step = 256 MiB worth of fresh uniform-random distinct row IDs of the config-4 host buffer read
at row width R from byte offset B -> dgz_order_ids + dgz_gather_perm (the product path for an
arbitrary ID list).

Metric: gathered feature GB/s (useful bytes n*R / time, GB = 1e9), whole-job aggregate over ranks.
Inputs are resident (CSR, seeds / ID lists in HBM, table pinned) before the timed region; the
56.9 GB table and fresh minibatches / ID lists every step are far larger than the 126 MB L2.
Rank 0 prints ONE JSON line.  ``--impl reference`` times the CPU oracle (oracle/, plain
single-threaded C) on the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import os
import resource
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
SWEEP_BYTES = 256 << 20            # config 5: bytes of rows per step
FORCE_MEMFD = os.environ.get("DGZ_BENCH_FORCE_MEMFD") == "1"   # tests: share host objects by memfd


# ----------------------------------------------------------------------------------------------
# distributed plumbing
# ----------------------------------------------------------------------------------------------
class Dist:
    def __init__(self, want_gpus: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        self.backend = None
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

    def gather_obj(self, obj):
        """Every rank's object, in rank order (all_gather_object; off the data path)."""
        if not self.pg:
            return [obj]
        out = [None] * self.world
        self.pg.all_gather_object(out, obj)
        return out

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
# preflight and host placement
# ----------------------------------------------------------------------------------------------
class PreflightError(RuntimeError):
    pass


def _meminfo_bytes(key: str) -> int | None:
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith(key + ":"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def preflight(d: Dist, shared_bytes: int, per_rank_bytes: int) -> dict:
    """Check, before anything is allocated, that the host can hold what this run maps: the shared
    table (+ CSR) in /dev/shm when N > 1 (a short tmpfs means SIGBUS on first touch, not an error),
    free RAM for it plus every rank's pinned staging, and the memlock limit for pinning.  Rank 0
    checks the shared objects; every rank checks its own memlock.  Raises PreflightError."""
    info, problems = {}, []
    if d.rank == 0:
        avail = _meminfo_bytes("MemAvailable")
        need_ram = shared_bytes + per_rank_bytes * d.world
        info.update(mem_available_gb=round(avail / 1e9, 1) if avail else None, need_ram_gb=round(need_ram / 1e9, 1))
        if avail is not None and avail < need_ram:
            problems.append(f"host RAM: {avail / 1e9:.1f} GB available < {need_ram / 1e9:.1f} GB needed "
                            f"({shared_bytes / 1e9:.1f} GB table/CSR + {d.world} x {per_rank_bytes / 1e9:.1f} GB per rank)")
        if d.world > 1:   # a short /dev/shm is not fatal: the shared objects then live in memfds (shared_host_name)
            st = os.statvfs("/dev/shm")
            free = st.f_bavail * st.f_frsize
            info["dev_shm_free_gb"] = round(free / 1e9, 1)
            info["shared_objects"] = "/dev/shm" if free >= shared_bytes else "memfd of rank 0 (/dev/shm too small)"
    soft, _ = resource.getrlimit(resource.RLIMIT_MEMLOCK)
    lim_ok = soft == resource.RLIM_INFINITY or soft >= shared_bytes or os.geteuid() == 0
    info["memlock"] = "unlimited" if soft == resource.RLIM_INFINITY else soft
    if not lim_ok:
        problems.append(f"rank {d.rank}: RLIMIT_MEMLOCK {soft} B < {shared_bytes} B to pin (ulimit -l unlimited)")
    allp = [p for ps in d.gather_obj(problems) for p in ps]
    if allp:
        raise PreflightError("; ".join(allp))
    return info


def _parse_cpulist(s: str) -> list:
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_numa_node(dev: int) -> int:
    """NUMA node of the GPU's PCIe function (sysfs), -1 when unknown."""
    try:
        p = torch.cuda.get_device_properties(dev)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            return int(f.read().strip())
    except Exception:
        return -1


def node_cpus(node: int) -> list:
    allowed = sorted(os.sched_getaffinity(0))
    if node < 0:
        return allowed
    try:
        with open(f"/sys/devices/system/node/node{node}/cpulist") as f:
            cpus = [c for c in _parse_cpulist(f.read()) if c in set(allowed)]
        return cpus or allowed
    except OSError:
        return allowed


def rank_cpu_share(d: Dist) -> tuple:
    """(this rank's host cores for CPU work, its GPU's NUMA node): the cores of the GPU's NUMA node,
    split evenly among the ranks whose GPUs sit on that node (all ranks when unknown)."""
    node = gpu_numa_node(torch.cuda.current_device())
    nodes = d.gather_obj(node)
    peers = [r for r, n in enumerate(nodes) if n == node]
    cpus = node_cpus(node)
    k = max(1, len(cpus) // len(peers))
    i = peers.index(d.rank)
    mine = cpus[i * k:(i + 1) * k] or cpus[:1]
    return mine, node


class pinned_threads:
    """Pin every thread of this process (torch's intra-op pool included) to `cpus`; restore on exit."""

    def __init__(self, cpus):
        self.cpus = set(cpus)

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        self.prev_threads = torch.get_num_threads()
        torch.set_num_threads(len(self.cpus))
        self._apply(self.cpus)
        return self

    @staticmethod
    def _apply(cpus):
        for tid in os.listdir("/proc/self/task"):
            try:
                os.sched_setaffinity(int(tid), cpus)
            except OSError:
                pass

    def __exit__(self, *a):
        self._apply(self.prev)
        torch.set_num_threads(self.prev_threads)


def sweep_buffer_cfg(args):
    """Config 5's host buffer: the config-4 table (56.9 GB) unless --table-gb shrinks it (tests)."""
    import dataclasses
    c4 = gen.CONFIGS[4]
    gb = getattr(args, "table_gb", 0.0)
    return dataclasses.replace(c4, n_nodes=int(gb * 1e9) // c4.row_bytes) if gb else c4


def workload_name(args) -> str:
    """The workload string both arms print (identical for the same flags)."""
    if args.config == 5:
        c4 = sweep_buffer_cfg(args)
        return (f"config5 row-width sweep: {args.row_bytes} B rows ({args.dtype}) at base offset {args.base} B of the "
                f"{c4.table_bytes / 1e9:.1f} GB config-4 host buffer, {SWEEP_BYTES >> 20} MiB of fresh uniform-random "
                "distinct rows per GPU per step")
    c = gen.CONFIGS[args.config]
    skew = f", power-law endpoints (alpha {args.skew_alpha})" if args.cache_frac > 0 else ""
    cache = f", {args.cache_frac:.0%} of rows cached in HBM (sharded over the GPUs)" if args.cache_frac > 0 else ""
    return (f"config{c.cid} {c.name}: {c.n_nodes} nodes (Poisson avg deg {c.avg_degree}{skew}), {c.dim}x fp32 = "
            f"{c.row_bytes} B rows, {c.table_bytes / 1e9:.1f} GB pinned host table, fanouts {list(c.fanouts)}, "
            f"{c.batch} seeds per GPU per step{cache}")


# ----------------------------------------------------------------------------------------------
# shared inputs
# ----------------------------------------------------------------------------------------------
def shared_host_name(d: Dist, nbytes: int, tag: str):
    """(name, fd to close after every rank mapped it) of a shared host object of `nbytes`: a /dev/shm
    object when /dev/shm can hold it, else a memfd of rank 0 that the other ranks open through
    /proc/<pid>/fd/<n> (shmem like /dev/shm, but not limited by the mount's size).  Collective."""
    name, fd = None, None
    if d.rank == 0:
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize >= nbytes + (256 << 20) and not FORCE_MEMFD:
            name = f"/dgz_bench_{tag}_{os.environ.get('MASTER_PORT', '0')}"
        else:
            fd = os.memfd_create(f"dgz_{tag}", 0)
            os.ftruncate(fd, nbytes)
            name = f"/proc/{os.getpid()}/fd/{fd}"
    return d.bcast_obj(name), fd


HOST_TABLE_POLICY = {
    "managed": "DGZ_HOST_MANAGED: cudaMallocManaged, preferred location CPU (filled in place by the CPU, never "
               "migrates), AccessedBy the GPU at registration; one copy per rank",
    "registered": "/dev/shm object shared by the ranks (NUMA-interleaved), cudaHostRegister'd by every rank"}


def host_table_kind(args, d: Dist, nbytes: int) -> str:
    """'managed' (DGZ_HOST_MANAGED: CUDA managed memory kept in host memory, mapped for the GPU with
    large pages -- DESIGN.md 5.1) or 'registered' (the paper's cudaHostRegister'd table, one shared
    /dev/shm copy per box).  auto: managed for one process; registered for N > 1 ranks
    (managed memory is not shareable across processes, and two processes allocating a 57 GB managed
    table each on one box failed in cudaMallocManaged here) -- `--host-table managed` forces one copy
    per rank."""
    kind = args.host_table
    if kind == "auto":
        kind = "managed" if d.world == 1 else "registered"
    return kind


def make_table(cfg, d: Dist, dgz, kind: str = "registered"):
    """Host feature table.  registered: one copy on the box, registered by every rank;
    managed: one DGZ_HOST_MANAGED copy per rank, filled in place by the CPU."""
    nbytes = cfg.table_bytes
    if kind == "managed":
        buf = dgz.HostBuffer(nbytes + 4096, flags=dgz.HOST_MANAGED)
        t0 = time.time()
        gen.fill_table(buf.ptr, nbytes, cfg.seed)
        return buf, time.time() - t0
    return make_registered_table(cfg, d, dgz)


def make_table_kind(cfg, d: Dist, dgz, kind: str):
    """make_table, falling back to the registered table when a managed allocation fails (N = 1 only:
    with N > 1 every rank must use the same kind).  Returns (buffer, fill seconds, kind used)."""
    if kind == "managed" and d.world == 1:
        try:
            buf, fill_s = make_table(cfg, d, dgz, "managed")
            return buf, fill_s, "managed"
        except Exception as e:   # DgzError from cudaMallocManaged / cudaMemAdvise
            print(f"# managed host table unavailable ({str(e)[:160]}); using the registered table", file=sys.stderr)
            buf, fill_s = make_table(cfg, d, dgz, "registered")
            return buf, fill_s, "registered (managed allocation failed)"
    buf, fill_s = make_table(cfg, d, dgz, kind)
    return buf, fill_s, kind


def make_registered_table(cfg, d: Dist, dgz):
    nbytes = cfg.table_bytes
    if d.world == 1:
        buf = dgz.HostBuffer(nbytes + 4096, flags=dgz.HOST_HUGEPAGE)
        t0 = time.time()
        gen.fill_table(buf.ptr, nbytes, cfg.seed)
        fill_s = time.time() - t0
    else:
        name, fd = shared_host_name(d, nbytes + 4096, f"c{cfg.cid}")
        fill_s = 0.0
        if d.rank == 0:   # interleaved over the sockets' memory when the box has several NUMA nodes
            buf = dgz.HostBuffer(nbytes + 4096, shm_name=name, create=fd is None,
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
            if fd is not None:
                os.close(fd)
    return buf, fill_s


def make_csr(cfg, d: Dist, dgz, skew_alpha: float = 0.0):
    """The graph's CSR on the host: plain arrays for N = 1; for N > 1 rank 0 generates it once
    into shared /dev/shm mappings that every rank maps (one host copy per box, not one per rank).
    Returns (offsets int64 view, cols int32 view, n_edges, keep-alive buffers)."""
    if d.world == 1:
        off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed, skew_alpha=skew_alpha)
        return off, col, int(off[-1]), []
    bufs, names, fds = [], [], []
    e = None
    if d.rank == 0:
        def alloc(nb):   # rank 0 only: a /dev/shm object, or a memfd when /dev/shm is short
            st = os.statvfs("/dev/shm")
            if st.f_bavail * st.f_frsize >= nb + (256 << 20) and not FORCE_MEMFD:
                name, fd = f"/dgz_bench_csr{cfg.cid}_{os.environ.get('MASTER_PORT', '0')}_{len(bufs)}", None
            else:
                fd = os.memfd_create(f"dgz_csr{len(bufs)}", 0)
                os.ftruncate(fd, nb + 4096)
                name = f"/proc/{os.getpid()}/fd/{fd}"
                fds.append(fd)
            b = dgz.HostBuffer(nb + 4096, shm_name=name, create=fd is None, flags=dgz.HOST_NUMA_INTERLEAVE)
            bufs.append(b)
            names.append(name)
            return b.ptr
        gen.set_threads(os.cpu_count() or 1)
        _, _, e = gen.gen_csr_into(cfg.n_nodes, cfg.avg_degree, cfg.seed, alloc, skew_alpha=skew_alpha)
        gen.set_threads(max(1, (os.cpu_count() or 1) // d.world))
    e, names = d.bcast_obj((e, names))
    e = int(e)
    if d.rank != 0:
        for name, nb in zip(names, ((cfg.n_nodes + 1) * 8, max(e * 4, 1))):
            bufs.append(dgz.HostBuffer(nb + 4096, shm_name=name, create=False))
    d.barrier()
    if d.rank == 0:
        for b in bufs:
            b.unlink()
        for fd in fds:
            os.close(fd)
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
    rtt = measure_rtt(dgz, pbuf, ptab)
    ptab.unregister()
    pbuf.free()
    del dbuf
    return {"h2d_dma_gbs": round(dma, 2), "h2d_dma_trials": [round(x, 2) for x in trials], "zc_stream_gbs": round(zc, 2),
            "ranks": d.world, "h2d_dma_aggregate_gbs": round(max(agg), 2), "zc_stream_aggregate_gbs": round(zc_agg, 2),
            "rtt": rtt,
            "how": "every rank at once after a barrier: best of 8 x (cudaMemcpyAsync 256 MiB pinned H2D x10) after 40 "
                   "warm-up copies; zero-copy "
                   "LDG.128 stream over a 1 GiB pinned buffer x4 on 8 SMs; aggregate = sum bytes / max time over ranks"}


def measure_rtt(dgz, pbuf, ptab, hops: int = 1000):
    """Round trip of one dependent zero-copy load (the Little's-law input): a pointer chase
    by one thread through the pinned buffer, (a) over 128 B lines inside 64 KiB regions already
    translated (the PCIe round trip), (b) one hop per fresh 64 KiB region (round trip + page walk).
    Cycles per hop at the SM clock; ns at the max SM clock of MEASURED_PEAKS.json."""
    arr = pbuf.numpy().view(np.int64)
    mhz = 1965.0
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
    except Exception:
        pass
    out = {}
    rng = np.random.default_rng(7)
    cyc = torch.zeros(2, dtype=torch.int64, device="cuda")
    for name, stride, base, m in (("in_region", 128, 0, 512), ("new_region", 65536, 64 << 20, hops)):
        slots = base // 8 + np.arange(m, dtype=np.int64) * (stride // 8)   # m nodes of one cycle
        order = rng.permutation(m)
        if name == "in_region":
            order = np.concatenate([[0], order[order != 0]])   # the chase starts at element 0
        for k in range(m):     # values are element indices from the buffer start (the chase's p)
            arr[slots[order[k]]] = slots[order[(k + 1) % m]]
        if name == "new_region":
            arr[0] = slots[order[0]]                             # element 0 -> the first fresh region
        if name == "in_region":     # one 64 KiB region: translate it once, then time the round trips
            dgz.probe_chase(ptab.info.dev_ptr, m, cyc)
        torch.cuda.synchronize()
        dgz.probe_chase(ptab.info.dev_ptr, hops, cyc)
        torch.cuda.synchronize()
        c = cyc[0].item() / hops
        out[name] = {"cycles": round(c, 1), "us_at_max_clock": round(c / mhz, 3)}
    out["how"] = "dgz_probe_chase: one thread, dependent ld.global.cv over the pinned buffer, 1000 hops"
    return out


def hbm_peak() -> float:
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling
    guide's fallback 6650 GB/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


TRAFFIC_FILES = ("profiles/r02/ncu_gather_summary.json", "profiles/r01/ncu_gather_summary.json")


def load_profile_traffic(key):
    """(dram bytes per gather launch, summary, source file) from the newest committed ncu --set full
    capture (a separate run of the same workload, not the timed launches)."""
    for rel in TRAFFIC_FILES:
        try:
            with open(os.path.join(ROOT, rel)) as f:
                c = json.load(f).get(key)
        except Exception:
            continue
        if c:
            return int(c["dram_bytes_per_launch"]), {k: v for k, v in c.items() if k != "launches"}, rel
    return None, None, None


def pct(xs, q):
    return round(float(np.percentile(xs, q)), 4)


def clocks_ok_note(clocks):
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(clocks.get("reasons") or [])
    return sorted(bad)


# ----------------------------------------------------------------------------------------------
# our implementation, configs 1-4: sample + gather per minibatch
# ----------------------------------------------------------------------------------------------
def run_ours(args, d: Dist):
    from paper_2103_03330_b200 import dgz
    from paper_2103_03330_b200.pipeline import MinibatchFetcher, calibrated_fetcher

    cfg = gen.CONFIGS[args.config]
    R = cfg.row_bytes
    G, rank = d.world, d.rank
    csr_bytes = (cfg.n_nodes + 1) * 8 + int(cfg.n_nodes * cfg.avg_degree * 1.01) * 4
    bound = gen.sample_bound(cfg.n_nodes, cfg.batch, cfg.fanouts)[-1]
    tkind = host_table_kind(args, d, cfg.table_bytes)
    per_rank_tab = cfg.table_bytes if tkind == "managed" else 0
    pre = preflight(d, (cfg.table_bytes if tkind == "registered" else 0) + csr_bytes,
                    2 * bound * R + (3 << 30) + (csr_bytes if G == 1 else 0) + per_rank_tab)
    t_setup = time.time()
    gen.set_threads(max(1, (os.cpu_count() or 1) // G))
    buf, fill_s, tkind = make_table_kind(cfg, d, dgz, tkind)
    d.barrier()
    table = dgz.register_table(buf.ptr, cfg.n_nodes, cfg.dim, dgz.F32)
    info = table.info
    t0 = time.time()
    off, col, n_edges, csr_bufs = make_csr(cfg, d, dgz, skew_alpha=args.skew_alpha if args.cache_frac > 0 else 0.0)
    csr_s = time.time() - t0
    if args.csr == "host":    # zero-copy CSR (NEXT-3): the sampler reads the host arrays over PCIe
        if tkind == "managed":   # the columns in managed host memory too (2 MiB GPU pages)
            graph = dgz.HostGraph(off, col, managed=True)
        else:
            graph = dgz.HostGraph(off.ctypes.data, col.ctypes.data, cfg.n_nodes, n_edges, False)
    else:                     # CSR replicated in each GPU's HBM
        graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())

    K, W = args.steps, args.warmup
    batches = [i * G + rank for i in range(W + K)]
    seeds_host = [torch.from_numpy(gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j)) for j in batches]
    seeds_dev = [x.cuda() for x in seeds_host]
    rng = [gen.batch_rng_seed(cfg.seed, j) for j in batches]

    cache, cache_info = None, None
    if args.cache_frac > 0:   # NEXT-1: hot rows = highest in-degree, cached in HBM, shard g on rank g
        assert args.csr == "hbm", "--cache-frac ranks rows by in-degree from the HBM CSR"
        k_hot = int(cfg.n_nodes * args.cache_frac)
        order = torch.argsort(torch.bincount(graph.cols.long(), minlength=cfg.n_nodes), descending=True)
        hot = order[:k_hot].contiguous()
        del order
        t0 = time.time()
        cache = dgz.ShardedHotRowCache(table, hot) if G > 1 else dgz.HotRowCache(table, hot, 1)
        torch.cuda.synchronize()
        cache_info = {"fraction": args.cache_frac, "rows": k_hot, "gb_total": round(k_hot * R / 1e9, 2),
                      "gb_per_gpu": round(k_hot * R / G / 1e9, 2), "shards": G, "fill_s": round(time.time() - t0, 2)}
        del hot

    gflags = dgz.FLAG_DYNAMIC if args.dynamic else 0
    gcfg = (dgz.gather_cfg(sm_count=args.gather_sms, warps_per_cta=args.gather_warps, flags=gflags)
            if (args.gather_sms or args.gather_warps or gflags) else None)
    choice = None
    if args.sampler_sms is None and not args.graphs and args.csr == "hbm":
        # the pipeline's shape is picked by measurement on the warm-up minibatches, before the timed
        # region (pipeline.calibrated_fetcher)
        fetcher, choice = calibrated_fetcher(table, graph, cfg.fanouts, cfg.batch, seeds_dev[:W], rng[:W], slots=2,
                                             gather_cfg=gcfg, blocks=True, cache=cache)
    else:
        fetcher = MinibatchFetcher(table, graph, cfg.fanouts, cfg.batch, slots=2, gather_cfg=gcfg, blocks=True,
                                   sampler_sms=args.sampler_sms, graphs=args.graphs, cache=cache)
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
        n = ns[i - W]
        last[batches[i]] = (mbs[i].bufs.ids[:n].cpu().numpy(), mbs[i].rows[:n].cpu().numpy(), rng[i],
                            seeds_host[i].numpy())

    # ---- cache statistics of the timed minibatches (re-sampled: the sampler is deterministic)
    cache_stats = None
    if cache is not None:
        cache_stats = run_cache_stats(dgz, cache, graph, cfg, seeds_dev, rng, W, K, G, rank, elapsed, gather_ms, ns, d)
        cache_info.update(cache_stats.pop("job"))

    # ---- end-to-end through the public API: pinned host seeds -> H2D -> sample -> gather -> D2H |U|
    e2e = run_e2e(fetcher, cfg, seeds_host, rng, W, K, d)

    # ---- minibatch-fetch latency, unpipelined: sampling then gather of one minibatch on one stream
    lat = run_latency(fetcher, cfg, seeds_dev, rng, min(K, 16), cache)

    # ---- overlap with a stand-in consumer (steps a5-a7); rank 0 (the others wait at the barrier)
    overlap = (run_overlap(dgz, fetcher, cfg, seeds_dev, rng, W, K, args)
               if (args.overlap and rank == 0 and cache is None) else None)
    d.barrier()

    # ---- baselines: the paper's DMA method (every rank), the oracle (rank 0, one core) + parity
    cpu_base = dma_base = parity = None
    cpus, node = rank_cpu_share(d)
    if not args.no_baselines:
        bt = baseline_table(dgz, buf, cfg.table_bytes, cfg.seed, tkind.startswith("managed") and G == 1)
        dma_base = run_dma_baseline(cfg, bt.buf, fetcher, seeds_dev, rng, K, d, cpus, node)
        dma_base["host_table"] = bt.what
        bt.close()
        if rank == 0:
            cpu_base, parity = run_oracle_leg(cfg, buf.ptr, off, col, last, d, cpus[0], budget=args.oracle_budget)
    all_in_gpu = None
    if G == 1 and not args.no_baselines and args.csr == "hbm" and cache is None:
        all_in_gpu = run_all_in_gpu(dgz, cfg, buf, graph, seeds_dev, rng, K)
    d.barrier()

    clocks = clk.summary()
    sm_count = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    tkey = (f"config{cfg.cid}" + ("_managed" if tkind == "managed" else "")
            + (f"_cache{args.cache_frac:g}" if cache is not None else ""))
    traffic, traffic_detail, traffic_src = load_profile_traffic(tkey)
    peak = ceilings["h2d_dma_gbs"]
    per_rank = d.gather_obj({"rank": rank, "device": torch.cuda.current_device(), "numa_node": node,
                             "register_s": round(info.register_seconds, 2), "step_gbs": round(per_gpu, 3),
                             "gather_gbs": round(gather_gbs, 3), "h2d_dma_gbs": peak,
                             "dma_baseline_gbs": dma_base["per_gpu_gbs"] if dma_base else None,
                             "host_cpus": f"{cpus[0]}-{cpus[-1]}" if cpus else None,
                             "pcie_bytes_avoided": cache_stats["pcie_bytes_avoided_rank"] if cache_stats else 0,
                             "peer_shard_bytes": cache_stats["peer_shard_bytes_rank"] if cache_stats else 0})
    kernel = "gather_segment_kernel (dgz_gather_perm)" if cache is None else "gather_segment_kernel CACHED (dgz_gather_cached)"
    if cache is not None:    # the link-bound part: missed rows over PCIe per gather launch
        ach = cache_stats["pcie_gbs_rank"]
    else:
        ach = gather_gbs
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": G, "steps": K, "warmup": W,
        "ms_per_step": round(max_el / K * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8 (fp32 rows moved as bytes)", "data": "synthetic",
        "config": {"workload": workload_name(args), "edges": n_edges,
                   "global_batch": cfg.batch * G, "parallelism": f"dp{G} (seed partition j mod G)",
                   "l2": "inputs larger than L2 (56.9 GB table, fresh minibatch every step)",
                   "pipeline": fetcher.mode, "pipeline_choice": choice,
                   "csr": "HBM (replicated per GPU)" if args.csr == "hbm" else
                          f"host memory ({'managed' if tkind == 'managed' else 'registered'}), sampled by zero-copy",
                   "host_table": tkind,
                   "gather": dict(dgz.gather_plan(table, cap, True, gcfg),
                                  order="address-sorted + inverse permutation (dgz_gather_perm)"),
                   "cache": cache_info},
        "per_gpu_gbs": round(per_gpu, 3),
        "roofline": {"bound": "pcie", "achieved": round(ach, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "traffic": traffic, "traffic_detail": traffic_detail,
                     "traffic_source": (f"ncu --set full capture of a separate run of this workload ({traffic_src}), "
                                        "dram__bytes_read.sum + dram__bytes_write.sum per gather launch; not the timed "
                                        "launches") if traffic_src else None,
                     "kernel": kernel,
                     "peak_source": "measured in this run: cudaMemcpyAsync H2D from pinned memory (PCIe Gen5 x16); "
                                    "MEASURED_PEAKS.json has no PCIe figure",
                     "algorithmic_bytes_per_launch": round(float(np.mean(ns)) * R),
                     "gather_ms_mean": round(float(np.mean(gather_ms)), 4),
                     "zc_stream_frac": round(ach / ceilings["zc_stream_gbs"], 4),
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
        "cpu_baseline": cpu_base, "dma_baseline": dma_base, "parity": parity, "cache_stats": cache_stats,
        "all_in_gpu": all_in_gpu,
        "e2e": e2e, "overlap": overlap, "per_rank": per_rank,
        "gpu_launches": int(launches), "gpu_launches_per_step": round(launches / K, 2),
        "clocks": clocks,
        "setup": {"table_fill_s": round(fill_s, 2), "register_s": round(info.register_seconds, 2),
                  "gpu_mem_mapping_bytes": info.gpu_mem_delta,
                  "mapping_ratio": round(cfg.table_bytes / max(info.gpu_mem_delta, 1), 1),
                  "csr_gen_s": round(csr_s, 2), "total_s": round(time.time() - t_setup, 1), "sms": sm_count,
                  "host_numa_nodes": dgz.host_numa_nodes(), "preflight": pre,
                  "host_table_policy": (HOST_TABLE_POLICY["managed"] if tkind == "managed" else
                                        HOST_TABLE_POLICY["registered"] if G > 1 else
                                        "anonymous THP mapping (first touch), cudaHostRegister")},
    }
    fetcher.close()
    if cache is not None and G > 1:
        cache.close()
    if args.csr == "host":
        graph.close()
    table.unregister()
    d.barrier()
    buf.free()
    for b in csr_bufs:
        b.free()
    return line


def run_cache_stats(dgz, cache, graph, cfg, seeds_dev, rng, W, K, G, rank, elapsed, gather_ms, ns, d: Dist):
    """Hit statistics of the timed minibatches: each is re-sampled (same seeds and sampler seed ->
    the same U) and its IDs looked up in the cache's slot map; shard owner = slot mod G."""
    R = cfg.row_bytes
    bufs = dgz.SampleBuffers(cfg.n_nodes, cfg.batch, cfg.fanouts, blocks=False, local=False)
    L = len(cfg.fanouts)
    hits = peer = rows = 0
    for i in range(W, W + K):
        dgz.sample_uniform(graph, seeds_dev[i], cfg.fanouts, rng[i], bufs)
        torch.cuda.synchronize()
        n = int(bufs.sizes_host[L])
        slot = cache.slot_map[bufs.ids[:n]]
        h = slot >= 0
        hits += int(h.sum())
        peer += int((h & (slot % G != rank)).sum())
        rows += n
    assert rows == sum(ns)
    miss = rows - hits
    t_g = sum(gather_ms) * 1e-3
    agg = d.allreduce([float(hits * R), float(peer * R), float(rows * R)], "sum")
    return {"hit_rate_rank": round(hits / max(rows, 1), 4), "peer_hit_rate_rank": round(peer / max(rows, 1), 4),
            "pcie_bytes_avoided_rank": hits * R, "peer_shard_bytes_rank": peer * R, "pcie_bytes_rank": miss * R,
            "pcie_gbs_rank": round(miss * R / t_g / 1e9, 3), "effective_gather_gbs_rank": round(rows * R / t_g / 1e9, 3),
            "peer_shard_gbs_rank": round(peer * R / t_g / 1e9, 3),
            "job": {"pcie_bytes_avoided_total": int(agg[0]), "peer_shard_bytes_total": int(agg[1]),
                    "hit_rate_total": round(agg[0] / max(agg[2], 1), 4)},
            "how": "timed minibatches re-sampled after the run (deterministic), IDs looked up in the slot map; "
                   "rates over the summed CUDA-event gather time of the timed launches"}


def run_latency(fetcher, cfg, seeds_dev, rng, n, cache=None):
    """Minibatch-fetch latency without pipelining: on one stream, sample (whole GPU) then gather,
    events around each phase; p10/p50/p90 over n fresh minibatches."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    f = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, sampler_sms=0, cache=cache)
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

    marks = []

    def loop(lo, hi):
        total, prev = 0, None
        for i in range(lo, hi):
            mb = fetcher.fetch(pinned[i], rng[i])
            if prev is not None:
                total += prev.sizes()[-1]
                marks.append(time.perf_counter())
            prev = mb
        return total + prev.sizes()[-1]
    loop(0, W)
    torch.cuda.synchronize()
    d.barrier()
    marks.clear()
    t0 = time.perf_counter()
    total = loop(W, W + K)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    gaps = np.diff([t0] + marks) * 1e3   # host-visible completion of step j-1, one per step
    tot, = d.allreduce([float(total * R)], "sum")
    mx, = d.allreduce([el], "max")
    L = len(cfg.fanouts)
    return {"value": round(tot / mx / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": cfg.batch * 8,
            "d2h_bytes_per_step": (L + 1) * 8, "ms_per_step": round(mx / K * 1e3, 4),
            "step_wall_ms_p10_p50_p90": [pct(gaps[1:], 10), pct(gaps[1:], 50), pct(gaps[1:], 90)] if len(gaps) > 2 else None,
            "pipeline": fetcher.mode,
            "how": "MinibatchFetcher.fetch(pinned host seeds) each step + host read of each step's |U| (one step "
                   "behind), wall clock, max over ranks"}


# default candidate shapes of the overlap leg's fetch partition: (SMs, spread over the GPCs?, warps per SM)
# and where the consumer runs: "partition" = the complementary green-context partition, "whole GPU" = a plain
# stream (its short-lived CTAs also fill the fetch partition's SMs)
OVERLAP_CANDIDATES = ((32, True, 2, "partition"), (24, True, 2, "partition"), (40, True, 2, "partition"),
                      (16, True, 4, "partition"), (48, True, 1, "partition"), (24, False, 2, "partition"),
                      (8, True, 8, "partition"),
                      (16, True, 4, "whole GPU"), (24, True, 2, "whole GPU"), (32, True, 2, "whole GPU"),
                      (48, True, 1, "whole GPU"), (64, True, 1, "whole GPU"), (74, True, 1, "whole GPU"))


def run_overlap(dgz, fetcher, cfg, seeds_dev, rng, W, K, args):
    """Exposed fetch time with a stand-in GraphSAGE mean-aggregation consumer (a5-a7) and the
    SM-partition sweep (a6; the B200 analogue of the paper's MPS ratio sweep, fig:mps_bandwidth):
    the fetch runs on a green-context partition of k SMs, the consumer on the other 148 - k, and
    step j+1 is fetched while step j is consumed.  Every candidate shape (SMs, spread or
    contiguous, warps per SM) and sampler placement is timed UNDER the consumer's load, the
    fastest overlapped step is reported as best, and its per-step timeline is recorded (CUDA
    events on each stream: sample, gather, consume)."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    dim = cfg.dim
    L = len(cfg.fanouts)
    nstep = min(K, 8)
    ev2 = (ev(), ev())

    hidden = args.consumer_hidden
    sage = args.consumer == "sage"   # any row width: wide rows (config 2, 602 fp32) are chunked along K
    # the layer's weight (nn.Linear layout [hidden, dim], bf16), seeded; only its shape matters for timing
    w_layer = (torch.randn(hidden, dim, generator=torch.Generator().manual_seed(7)) / dim ** 0.5).to(torch.bfloat16).cuda()

    cons_roof = {}

    def consume(comp, mb, repeat, y, nb, cb):
        torch.cuda.nvtx.range_push("dgz.consume")
        _consume(comp, mb, repeat, y, nb, cb)
        torch.cuda.nvtx.range_pop()

    def _consume(comp, mb, repeat, y, nb, cb):
        if sage:   # mean over the sampled neighbours, then the GEMM (tcgen05)
            dgz.sage_mean_linear(mb.rows.view(torch.float32).view(-1), dim, mb.bufs.local[nb:], mb.bufs.cnt[cb:],
                                 cfg.fanouts[L - 1], mb.bufs.sizes_dev[L - 1:L], mb.bufs.bounds[L - 1], w_layer, y,
                                 repeat=repeat, ctas_per_sm=args.consumer_ctas_per_sm, stream=comp)
        else:
            dgz.aggregate_mean(mb.rows.view(torch.float32).view(-1), dim, mb.bufs.local[nb:], mb.bufs.cnt[cb:],
                               cfg.fanouts[L - 1], mb.bufs.sizes_dev[L - 1:L], mb.bufs.bounds[L - 1], y, repeat=repeat,
                               stream=comp)

    def measure(f, comp, repeat=None, t_target=None, timeline=False):
        y = torch.empty((f.bufs[0].bounds[L - 1], hidden if sage else dim), dtype=torch.float32, device="cuda")
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
        calibrate = repeat is None
        if calibrate:
            repeat = 8
            for _ in range(3):
                repeat = max(1, int(round(repeat * (t_target or t_g) / cons_alone(repeat))))
        t_c = cons_alone(repeat)
        if calibrate:   # the consumer kernel's own roofline: algorithmic HBM bytes per launch / launch time
            n_dst = int(mb.sizes()[L - 1])
            c = mb.bufs.cnt[cb:cb + n_dst].to(torch.int64).cpu()
            f_last = cfg.fanouts[L - 1]
            byts = (int(c.sum()) + n_dst) * dim * 4 + n_dst * (4 + 4 * f_last) + n_dst * (hidden if sage else dim) * 4
            byts += hidden * dim * 2 if sage else 0
            ms = t_c / repeat
            peak = hbm_peak()
            cons_roof.update({"kernel": "sage_mean_linear_kernel" if sage else "aggregate_mean_kernel", "bound": "hbm",
                              "n_dst": n_dst, "launch_ms": round(ms, 4), "alg_bytes_per_launch": byts,
                              "achieved_gbs": round(byts / ms / 1e6, 1), "peak_gbs": peak,
                              "frac": round(byts / ms / 1e6 / peak, 3),
                              "gemm_tflops": round(2.0 * n_dst * dim * hidden / ms / 1e9, 2) if sage else None,
                              "how": "rows read (1 + cnt) x dim x 4 B + block (4 + 4 fanout) B + output row per dst node "
                                     "(+ W once), per launch = T_c / repeat alone on the whole GPU; peak = "
                                     "MEASURED_PEAKS.json hbm_gbs (else the guide's 6650)"})
        torch.cuda.synchronize()
        trace = []
        ahead = len(f.bufs) - 1   # minibatches fetched ahead of the one being consumed (slots - 1)
        mbs = [f.fetch(seeds_dev[i % len(rng)], rng[i % len(rng)], timing=timeline) for i in range(ahead)]
        a0 = ev()
        a0.record(comp)
        comp.wait_event(mbs[0].event)   # steady state: the pipeline's fill (the first fetch) is charged separately
        a.record(comp)
        for i in range(ahead, nstep + ahead):
            nxt = f.fetch(seeds_dev[i % len(rng)], rng[i % len(rng)], timing=timeline)
            cur = mbs.pop(0)
            comp.wait_event(cur.event)
            if timeline:
                c0, c1 = ev(), ev()
                c0.record(comp)
            consume(comp, cur, repeat, y, nb, cb)
            if timeline:
                c1.record(comp)
                trace.append((cur.timing, (c0, c1)))
            f.release(cur, comp)
            mbs.append(nxt)
        comp.wait_event(mbs[0].event)   # the next minibatch is fetched too (as with 2 slots)
        b.record(comp)
        torch.cuda.synchronize()
        t_o = a.elapsed_time(b) / nstep
        t_o_fill = a0.elapsed_time(b) / nstep
        tl = None
        if timeline:
            tl = []
            for k, ((s0, g0, g1), (c0, c1)) in enumerate(trace):
                tl.append({"step": k, "sample": [round(a.elapsed_time(s0), 3), round(a.elapsed_time(g0), 3)],
                           "gather": [round(a.elapsed_time(g0), 3), round(a.elapsed_time(g1), 3)],
                           "consume": [round(a.elapsed_time(c0), 3), round(a.elapsed_time(c1), 3)]})
        return t_g, t_c, t_o, repeat, tl, t_o_fill

    f0 = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, sampler_sms=0)
    comp0 = torch.cuda.Stream()
    t_g0, t_c0, t_o0, repeat, _, t_of0 = measure(f0, comp0)
    del f0
    rows = [{"partition": "none (whole GPU, high-priority fetch stream)", "fetch_sms": 148, "t_fetch_ms": round(t_g0, 3),
             "t_consumer_ms": round(t_c0, 3), "t_step_overlapped_ms": round(t_o0, 3),
             "t_step_overlapped_incl_fill_ms": round(t_of0, 3), "exposed_fetch_ms": round(max(0.0, t_o0 - t_c0), 3)}]
    cands = OVERLAP_CANDIDATES
    if args.overlap_warps:
        cands = tuple((k, sp, args.overlap_warps, c) for k, sp, _, c in cands)
    def build(k, spread, w, where, cons):
        """Partitions + fetcher of one shape: the gather on k SMs (spread over the GPCs or contiguous),
        the sampler in front of it, in the consumer's stream, or on its own 8-SM partition (explicit SM
        groups disjoint from the gather's, so sampling j+1 overlaps gathering j), the consumer on the
        complementary partition or on the whole GPU (a plain stream)."""
        parts = []
        if where == "own 8-SM partition":
            ng, per = dgz.partition_groups()
            m = max(1, -(-k // per))
            gg = [i * ng // m for i in range(m)]
            rest = [g for g in range(ng) if g not in set(gg)]
            ms = max(1, -(-8 // per))
            sg = [rest[i * len(rest) // ms] for i in range(ms)]
            parts = [dgz.Partition(0, -1, 0, groups=gg), dgz.Partition(0, -1, 0, groups=sg)]
            gpart, sstream = parts[0], parts[1].fetch_stream
        else:
            parts = [dgz.Partition(k, -1, dgz.PARTITION_SPREAD if spread else 0)]
            gpart, sstream = parts[0], None
            if where == "fetch partition, own stream":   # sampling j+1 beside gathering j on the same SMs
                sstream = gpart.stream(0, -1)
            elif where == "own stream":   # a high-priority stream of the primary context: the whole GPU, beside the consumer
                sstream = torch.cuda.Stream(priority=-1)
        comp = gpart.compute_stream if cons == "partition" else comp0
        if where == "consumer stream":
            sstream = comp
        pcfg = dgz.gather_cfg(sm_count=gpart.fetch_sms, warps_per_cta=w, flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)
        f = MinibatchFetcher(fetcher.table, fetcher.graph, cfg.fanouts, cfg.batch, fetch_stream=gpart.fetch_stream,
                             gather_cfg=pcfg, sample_stream=sstream, slots=args.overlap_slots)
        return f, comp, parts, gpart

    for k, spread, w, placement in cands:
        shape = "spread over the GPCs" if spread else "contiguous"
        # work-counter batches (a partition's slower SMs take fewer batches, explore28), 16 line loads per
        # lane, few warps per SM: beside a DRAM-heavy consumer the page walks slow down and fewer rows in
        # flight win.  Sampler placement x consumer placement, all measured.
        combos = ((("fetch partition", "partition"), ("fetch partition, own stream", "partition"),
                   ("consumer stream", "partition")) if placement == "partition"
                  else (("fetch partition", "whole GPU"), ("fetch partition, own stream", "whole GPU"),
                        ("consumer stream", "whole GPU"), ("own stream", "whole GPU"), ("own 8-SM partition", "whole GPU")))
        for where, cons in combos:
            if where == "own 8-SM partition" and not spread:
                continue
            try:
                f, comp, parts, gpart = build(k, spread, w, where, cons)
            except Exception as e:  # green contexts unavailable: report and skip
                rows.append({"fetch_sms": k, "error": str(e)[:200]})
                continue
            t_g, t_c, t_o, _, _, t_of = measure(f, comp, repeat=repeat)
            rows.append({"partition": f"green context ({shape}), sampler in the {where}, consumer on the "
                                      + ("other SMs" if cons == "partition" else "whole GPU"),
                         "fetch_sms": gpart.fetch_sms, "warps_per_sm": w,
                         "compute_sms": gpart.compute_sms if cons == "partition" else 148,
                         "t_fetch_ms": round(t_g, 3), "t_consumer_ms": round(t_c, 3), "t_step_overlapped_ms": round(t_o, 3),
                         "t_step_overlapped_incl_fill_ms": round(t_of, 3),
                         "exposed_fetch_ms": round(max(0.0, t_o - t_c0), 3),
                         "exposed_vs_own_sms_ms": round(max(0.0, t_o - t_c), 3),
                         "fetch_gbs_alone": round(float(f.bufs[0].sizes_host[-1]) * cfg.row_bytes / t_g / 1e6, 2),
                         "shape": [k, spread, w, where, cons]})
            del f
            torch.cuda.synchronize()
            for pt in parts:
                pt.destroy()
    # T_c on the whole GPU = the median of every whole-GPU consumer-alone measurement of the leg (the first
    # one alone drifts by up to ~8 % with clocks); exposed fetch = overlapped step - T_c
    tcs = [t_c0] + [r["t_consumer_ms"] for r in rows if "shape" in r and r["shape"][4] == "whole GPU"]
    t_c0 = float(np.median(tcs))
    for r in rows:
        if "t_step_overlapped_ms" in r:
            r["exposed_fetch_ms"] = round(max(0.0, r["t_step_overlapped_ms"] - t_c0), 3)
    # best = the shortest overlapped step (exposed fetch = overlapped step - the consumer alone on the whole
    # GPU, so the shortest step is also the least exposed fetch)
    best = min((r for r in rows if "t_step_overlapped_ms" in r), key=lambda r: r["t_step_overlapped_ms"])
    # round 1's definition, kept for comparison: the shortest step among shapes whose consumer is confined to
    # the complementary partition, exposed against that consumer alone on its own SMs
    part_rows = [r for r in rows if "shape" in r and r["shape"][4] == "partition"]
    hidden_partitioned = None
    if part_rows:
        bp = min(part_rows, key=lambda r: r["t_step_overlapped_ms"])
        hidden_partitioned = {"value": round(1 - bp["exposed_vs_own_sms_ms"] / t_g0, 3), "shape": bp["shape"],
                              "t_step_overlapped_ms": bp["t_step_overlapped_ms"], "t_consumer_own_sms_ms": bp["t_consumer_ms"]}
    timeline = None
    if "shape" in best:   # the best shape again, with per-step events on every stream
        k, spread, w, where, cons = best["shape"]
        f, comp, parts, gpart = build(k, spread, w, where, cons)
        t_g, t_c, t_o, _, tl, _ = measure(f, comp, repeat=repeat, timeline=True)
        del f
        torch.cuda.synchronize()
        for pt in parts:
            pt.destroy()
        timeline = {"shape": {"fetch_sms": k, "spread": spread, "warps_per_sm": w, "sampler": where, "consumer": cons},
                    "t_step_overlapped_ms": round(t_o, 3), "steps": tl,
                    "how": "CUDA events around each phase on its own stream, ms from the first consumer step's start"}
        if args.timeline:
            write_chrome_trace(args.timeline, timeline)
    return {"t_fetch_ms": round(t_g0, 3), "consumer_repeat": repeat, "t_consumer_ms": round(t_c0, 3),
            "t_consumer_samples_ms": [round(x, 3) for x in tcs], "consumer_roofline": cons_roof,
            "serial_ms": round(t_g0 + t_c0, 3), "best": best,
            "hidden_frac_best": round(1 - best["exposed_fetch_ms"] / t_g0, 3),
            "hidden_frac_partitioned": hidden_partitioned,
            "hidden_frac_best_incl_fill": round(1 - max(0.0, best["t_step_overlapped_incl_fill_ms"] - t_c0) / t_g0, 3),
            "steps_measured": nstep, "sweep": rows, "timeline": timeline,
            "consumer": (f"dgz_sage_mean_linear (mean over the sampled neighbours, then the {dim} x {hidden} bf16 GEMM on the "
                         "tensor cores)" if sage else "dgz_aggregate_mean")
                        + " over the last hop's block, non-persistent launches, repeated to T_c ~ T_fetch",
            "partition_gather": "candidate shapes (SMs, spread/contiguous, warps per SM) timed under load, 16 loads per "
                                "lane, work-counter batches",
            "hidden": "hidden_frac_best = 1 - exposed / T_fetch for the shortest overlapped step, exposed = T_overlap - T_c "
                      "(SURVEY 8(a) a7) with T_fetch and T_c each ALONE on the whole GPU, i.e. the share of the serial "
                      "step's fetch time that overlap removes; hidden_frac_partitioned = round 1's definition (the "
                      "shortest step among shapes whose consumer is confined to the other SMs, T_c = that consumer alone "
                      "on those SMs: larger whenever confinement slows the consumer); steady state: from the first "
                      "consumer step's start (the pipeline's first fetch, the fill, is in the *_incl_fill keys)"}


def write_chrome_trace(path, timeline):
    """The overlap timeline as a Chrome trace (chrome://tracing / Perfetto): one track per stream."""
    evs = []
    tid = {"sample": 1, "gather": 2, "consume": 3}
    for s in timeline["steps"]:
        for k in ("sample", "gather", "consume"):
            a, b = s[k]
            evs.append({"name": f"{k} {s['step']}", "ph": "X", "pid": 0, "tid": tid[k], "ts": a * 1e3, "dur": (b - a) * 1e3})
    for k, t in tid.items():
        evs.append({"name": "thread_name", "ph": "M", "pid": 0, "tid": t, "args": {"name": k}})
    os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
    with open(path, "w") as f:
        json.dump({"traceEvents": evs, "otherData": {"shape": timeline["shape"]}}, f)


def run_oracle_leg(cfg, table_addr, off, col, last, d: Dist, core: int, budget: float = 20.0):
    """cpu_baseline: the oracle as it stands (single-threaded C) on a bounded sample of the same
    workload (about `budget` seconds), on ONE core of GPU 0's NUMA node (sched_setaffinity), plus
    a full-size exact parity check of the GPU's last two minibatches."""
    import oracle
    R = cfg.row_bytes
    parity = {"batches": [], "exact": True}
    t_total, bytes_total, nb = 0.0, 0, 0
    prev = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {core})
    try:
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
    finally:
        os.sched_setaffinity(0, prev)
    return ({"value": round(bytes_total / t_total / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
             "sample": f"{nb} config{cfg.cid} minibatches (sample + gather, {t_total:.1f} s single-threaded C)",
             "s_per_minibatch": round(t_total / nb, 3), "host_cores": os.cpu_count(), "core": core,
             "ranks": d.world, "note": "rank 0 only, after the timed region, pinned to one core of its GPU's NUMA node"},
            parity)


def run_all_in_gpu(dgz, cfg, buf, graph, seeds_dev, rng, K):
    """Context only (the paper's All-in-GPU): the whole table copied
    into HBM once and fetched by the same sampler + gather kernels (frontier order, HBM-speed gather);
    the bound any host-memory method is compared against.  N = 1 only (one 56.9 GB HBM copy)."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    R = cfg.row_bytes
    dev = torch.empty(cfg.table_bytes, dtype=torch.uint8, device="cuda")
    dev.copy_(torch.from_numpy(buf.numpy(0, cfg.table_bytes)))      # registered pages: one DMA
    dtab = dgz.DeviceTable(dev.data_ptr(), cfg.n_nodes, cfg.dim, dgz.F32)
    f = MinibatchFetcher(dtab, graph, cfg.fanouts, cfg.batch, sampler_sms=0)
    nb = min(K, 8)
    for i in range(2):
        f.fetch(seeds_dev[i], rng[i])
    torch.cuda.synchronize()
    a, b = ev(), ev()
    mbs = []
    cnt = torch.zeros(nb, dtype=torch.int64, device="cuda")
    a.record(f.stream)
    for i in range(nb):
        mbs.append(f.fetch(seeds_dev[i], rng[i], timing=True, count_into=cnt[i:i + 1]))
    b.record(f.stream)
    torch.cuda.synchronize()
    g_ms = [mb.timing[1].elapsed_time(mb.timing[2]) for mb in mbs]
    el = a.elapsed_time(b) * 1e-3
    n_mean = float(cnt.double().mean())
    out = {"step_gbs": round(n_mean * R * nb / el / 1e9, 1), "gather_gbs": round(n_mean * R / (float(np.mean(g_ms)) * 1e-3) / 1e9, 1),
           "ms_per_step": round(el / nb * 1e3, 3), "gather_ms": round(float(np.mean(g_ms)), 3),
           "hbm_traffic_frac": round(2 * n_mean * R / (float(np.mean(g_ms)) * 1e-3) / 1e9 / hbm_peak(), 3),
           "how": "table copied to HBM (dgz_wrap_device_table), same fetcher, sample then gather on one stream, "
                  f"{nb} minibatches (GB/s of useful bytes; HBM traffic = reads + writes of the rows)"}
    f.close()
    dtab.unregister()
    del dev
    torch.cuda.empty_cache()
    return out


def _chunked_dma(host_rows, ids_cpu, R, stage, dst, cs, done):
    """CPU gather (torch.index_select) into pinned staging in chunks, each chunk's cudaMemcpyAsync
    H2D overlapping the CPU gather of the next (double-buffered)."""
    n = ids_cpu.numel()
    per = max(1, stage[0].numel() // R)
    k = 0
    for c0 in range(0, n, per):
        p = k % 2
        done[p].synchronize()
        m = min(per, n - c0)
        st = stage[p][:m * R].view(m, R)
        torch.index_select(host_rows, 0, ids_cpu[c0:c0 + m], out=st)
        with torch.cuda.stream(cs):
            dst[c0 * R:(c0 + m) * R].view(m, R).copy_(st, non_blocking=True)
            done[p].record(cs)
        k += 1


class baseline_table:
    """The host table the CPU-gather baseline reads: the product's own table, except that a managed
    table (whose CPU mapping uses 4 KiB pages) is replaced, at N = 1, by a THP-backed anonymous copy with
    the same bytes when host RAM allows -- the baseline gets the best CPU-side layout this box offers."""

    def __init__(self, dgz, buf, nbytes: int, seed: int, managed: bool):
        self.buf, self.copy, self.what = buf, None, "the product's table"
        if managed and (_meminfo_bytes("MemAvailable") or 0) > nbytes + (16 << 30):
            self.copy = dgz.HostBuffer(nbytes + 4096, flags=dgz.HOST_HUGEPAGE)
            gen.fill_table(self.copy.ptr, nbytes, seed)
            self.buf, self.what = self.copy, "a THP anonymous copy of the table (same bytes)"

    def close(self):
        if self.copy is not None:
            self.copy.free()
            self.copy = None


def run_dma_baseline(cfg, buf, fetcher, seeds_dev, rng, K, d: Dist, cpus, node):
    """The paper's DMA-based method: CPU gathers the sampled rows into a pinned
    staging buffer with T threads, then cudaMemcpyAsync H2D; double-buffered so the CPU gather
    of j+1 overlaps the copy of j.  Same IDs as the GPU path (sampled on the GPU beforehand).
    Every rank at once, each on its share of its GPU's NUMA-node cores (threads pinned)."""
    R = cfg.row_bytes
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
    with pinned_threads(cpus):
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
    return {"value": round(tot / mx / 1e9, 3), "unit": UNIT, "threads_per_rank": len(cpus), "ranks": d.world,
            "numa_node": node, "cpus": f"{cpus[0]}-{cpus[-1]}", "minibatches_per_rank": nb,
            "per_gpu_gbs": round(total / el / 1e9, 3),
            "how": "paper's DMA-based method (P:650-651): torch.index_select into pinned staging (the GPU's NUMA-node cores "
                   "split among the ranks on that node, threads pinned) + cudaMemcpyAsync, double-buffered, all ranks "
                   "concurrently; aggregate = sum bytes / max time"}


# ----------------------------------------------------------------------------------------------
# our implementation, config 5: the row-width sweep point (product path on an arbitrary ID list)
# ----------------------------------------------------------------------------------------------
def sweep_ids(rows: int, n: int, rank: int, step: int, R: int, base: int) -> np.ndarray:
    return gen.distinct_ids(rows, n, (R * 1_000_003 + base * 7919 + rank * 104_729 + step) & (2**63 - 1))


def run_rowsweep(args, d: Dist):
    from paper_2103_03330_b200 import dgz

    c4 = sweep_buffer_cfg(args)
    R, base = args.row_bytes, args.base
    dtype = dgz.F16 if args.dtype == "f16" else dgz.F32
    eb = dgz.ELEM_BYTES[dtype]
    assert R % eb == 0 and base % eb == 0 and 0 <= base <= 4096 - 64, "row bytes / base must be element-aligned"
    G, rank = d.world, d.rank
    K, W = args.steps, args.warmup
    total = c4.table_bytes
    rows = (total - base) // R
    n = min(rows, SWEEP_BYTES // R)
    # per rank: the ID lists on the host and their pinned copies (e2e leg), DMA staging, ceilings' buffers
    tkind = host_table_kind(args, d, total)
    pre = preflight(d, total if tkind == "registered" else 0,
                    2 * (W + K) * n * 8 + 2 * (32 << 20) + (3 << 30) + (total if tkind == "managed" else 0))
    t_setup = time.time()
    gen.set_threads(max(1, (os.cpu_count() or 1) // G))
    buf, fill_s, tkind = make_table_kind(c4, d, dgz, tkind)
    d.barrier()
    table = dgz.register_table(buf.ptr + base, rows, R // eb, dtype)
    info = table.info
    ids_host = [torch.from_numpy(sweep_ids(rows, n, rank, i, R, base)) for i in range(W + K)]
    ids_dev = [x.cuda() for x in ids_host]
    orderer = dgz.Orderer(n)
    out = torch.empty(n * R + 64, dtype=torch.uint8, device="cuda")
    ceilings = measure_ceilings(dgz, d)
    s = torch.cuda.Stream(priority=-1)
    evs = [(ev(), ev(), ev()) for _ in range(W + K)]

    def step(i):
        a, g0, g1 = evs[i]
        a.record(s)
        srt, pos = orderer.order(ids_dev[i], rows, stream=s)
        g0.record(s)
        dgz.gather_perm(table, srt, pos, out, n=n, stream=s)
        g1.record(s)

    for i in range(W):
        step(i)
    torch.cuda.synchronize()
    d.barrier()
    torch.cuda.synchronize()
    launches0 = dgz.kernel_launches()
    t_start, t_end = ev(), ev()
    with ClockSampler(d.local) as clk:
        t_start.record(s)
        for i in range(W, W + K):
            step(i)
        t_end.record(s)
        torch.cuda.synchronize()
    launches = dgz.kernel_launches() - launches0
    d.barrier()
    dgz.check_errors(table)
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    gather_ms = [evs[i][1].elapsed_time(evs[i][2]) for i in range(W, W + K)]
    order_ms = [evs[i][0].elapsed_time(evs[i][1]) for i in range(W, W + K)]
    bytes_rank = float(K * n * R)
    tot_bytes, = d.allreduce([bytes_rank], "sum")
    max_el, = d.allreduce([elapsed], "max")
    value = tot_bytes / max_el / 1e9
    per_gpu = bytes_rank / elapsed / 1e9
    gather_gbs = n * R / (float(np.mean(gather_ms)) * 1e-3) / 1e9
    last = out[:n * R].cpu().numpy().reshape(n, R)
    last_ids = ids_host[W + K - 1].numpy()

    # ---- end to end: pinned host ID list -> H2D -> order -> gather -> D2H of the step's last 8 bytes
    pinned = [x.pin_memory() for x in ids_host]
    idx_stage = torch.empty(n, dtype=torch.int64, device="cuda")
    res = torch.empty(8, dtype=torch.uint8).pin_memory()

    def e2e_step(i):
        with torch.cuda.stream(s):
            idx_stage.copy_(pinned[i], non_blocking=True)
            srt, pos = orderer.order(idx_stage, rows, stream=s)
            dgz.gather_perm(table, srt, pos, out, n=n, stream=s)
            res.copy_(out[n * R - 8:n * R], non_blocking=True)
    for i in range(W):
        e2e_step(i)
    torch.cuda.synchronize()
    d.barrier()
    t0 = time.perf_counter()
    for i in range(W, W + K):
        e2e_step(i)
    s.synchronize()
    el = time.perf_counter() - t0
    etot, = d.allreduce([bytes_rank], "sum")
    emx, = d.allreduce([el], "max")
    e2e = {"value": round(etot / emx / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": 8,
           "ms_per_step": round(emx / K * 1e3, 4),
           "how": "pinned host ID list -> H2D -> dgz_order_ids -> dgz_gather_perm -> D2H of the result's last 8 bytes, "
                  "one stream, wall clock, max over ranks"}

    # ---- baselines: the paper's DMA method on the same lists (every rank), the oracle + parity (rank 0)
    cpus, node = rank_cpu_share(d)
    dma_base = cpu_base = parity = None
    if not args.no_baselines:
        bt = baseline_table(dgz, buf, total, c4.seed, tkind == "managed" and G == 1)
        host_rows = torch.from_numpy(bt.buf.numpy(base, rows * R)).view(rows, R)
        stage = [torch.empty(32 << 20, dtype=torch.uint8).pin_memory() for _ in range(2)]
        cs = torch.cuda.Stream()
        done = [torch.cuda.Event(), torch.cuda.Event()]
        nb = min(K, 4)
        with pinned_threads(cpus):
            _chunked_dma(host_rows, ids_host[W], R, stage, out, cs, done)
            torch.cuda.synchronize()
            d.barrier()
            t0 = time.perf_counter()
            for i in range(W, W + nb):
                _chunked_dma(host_rows, ids_host[i], R, stage, out, cs, done)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
        dt, = d.allreduce([float(nb * n * R)], "sum")
        dm, = d.allreduce([el], "max")
        del host_rows
        what = bt.what
        bt.close()
        dma_base = {"value": round(dt / dm / 1e9, 3), "unit": UNIT, "threads_per_rank": len(cpus), "ranks": G,
                    "host_table": what,
                    "numa_node": node, "per_gpu_gbs": round(nb * n * R / el / 1e9, 3), "lists_per_rank": nb,
                    "how": "torch.index_select into pinned staging (32 MiB chunks) + cudaMemcpyAsync, double-buffered, "
                           "threads pinned to the GPU's NUMA-node share, same ID lists, all ranks concurrently"}
        if rank == 0:
            cpu_base, parity = run_oracle_rowsweep(buf.ptr + base, rows, R, last_ids, last, ids_host, W, K, cpus[0],
                                                   args.oracle_budget, d)
    d.barrier()
    clocks = clk.summary()
    traffic, traffic_detail, traffic_src = load_profile_traffic(f"config5_R{R}_b{base}_{args.dtype}")
    peak = ceilings["h2d_dma_gbs"]
    per_rank = d.gather_obj({"rank": rank, "device": torch.cuda.current_device(), "numa_node": node,
                             "register_s": round(info.register_seconds, 2), "step_gbs": round(per_gpu, 3),
                             "gather_gbs": round(gather_gbs, 3), "h2d_dma_gbs": peak,
                             "dma_baseline_gbs": dma_base["per_gpu_gbs"] if dma_base else None})
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": G, "steps": K, "warmup": W,
        "ms_per_step": round(max_el / K * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": f"u8 ({args.dtype} rows moved as bytes)", "data": "synthetic",
        "config": {"workload": workload_name(args), "row_bytes": R, "base_offset": base, "elem": args.dtype, "rows": rows,
                   "rows_per_step": n, "parallelism": f"dp{G} (independent ID lists per rank)", "host_table": tkind,
                   "l2": "inputs larger than L2 (56.9 GB table, a fresh 256 MiB ID list every step)",
                   "gather": dict(dgz.gather_plan(table, n, True, None), order="dgz_order_ids + dgz_gather_perm")},
        "per_gpu_gbs": round(per_gpu, 3),
        "roofline": {"bound": "pcie", "achieved": round(gather_gbs, 3), "peak": peak, "unit": "GB/s",
                     "frac": round(gather_gbs / peak, 4), "traffic": traffic, "traffic_detail": traffic_detail,
                     "traffic_source": (f"ncu --set full capture of a separate run ({traffic_src})") if traffic_src else None,
                     "kernel": "gather_segment_kernel (dgz_gather_perm)",
                     "peak_source": "measured in this run: cudaMemcpyAsync H2D from pinned memory",
                     "algorithmic_bytes_per_launch": n * R, "gather_ms_mean": round(float(np.mean(gather_ms)), 4),
                     "order_ms_mean": round(float(np.mean(order_ms)), 4),
                     "zc_stream_frac": round(gather_gbs / ceilings["zc_stream_gbs"], 4),
                     "rows_per_s": round(n / (float(np.mean(gather_ms)) * 1e-3)),
                     "aggregate": {"achieved": round(value, 3), "peak": ceilings["h2d_dma_aggregate_gbs"],
                                   "frac": round(value / ceilings["h2d_dma_aggregate_gbs"], 4),
                                   "zc_peak": ceilings["zc_stream_aggregate_gbs"]}},
        "ceilings": ceilings, "cpu_baseline": cpu_base, "dma_baseline": dma_base, "parity": parity, "e2e": e2e,
        "per_rank": per_rank, "gpu_launches": int(launches), "gpu_launches_per_step": round(launches / K, 2),
        "clocks": clocks,
        "setup": {"table_fill_s": round(fill_s, 2), "register_s": round(info.register_seconds, 2),
                  "total_s": round(time.time() - t_setup, 1), "preflight": pre},
    }
    table.unregister()
    d.barrier()
    buf.free()
    return line


def run_oracle_rowsweep(table_addr, rows, R, last_ids, last_out, ids_host, W, K, core, budget, d: Dist):
    """Config 5 oracle leg: exact parity of the GPU's last full step (every row), then the oracle's
    gather timed on the same lists for about `budget` seconds, on one core."""
    import oracle
    prev = os.sched_getaffinity(0)
    os.sched_setaffinity(0, {core})
    try:
        n = last_ids.shape[0]
        want = np.empty(n * R, dtype=np.uint8)
        t0 = time.perf_counter()
        bad = oracle.gather_into(table_addr, rows, R, last_ids, want)
        t_total = time.perf_counter() - t0
        parity = {"rows": int(n), "rows_equal": bool(bad == 0 and np.array_equal(want.reshape(n, R), last_out)),
                  "what": "every row of the last timed step vs the oracle"}
        parity["exact"] = parity["rows_equal"]
        done, i = n, W
        while t_total < budget and i < W + K:
            ids = ids_host[i].numpy()
            t0 = time.perf_counter()
            oracle.gather_into(table_addr, rows, R, ids, want)
            t_total += time.perf_counter() - t0
            done += ids.shape[0]
            i += 1
    finally:
        os.sched_setaffinity(0, prev)
    return ({"value": round(done * R / t_total / 1e9, 4), "unit": UNIT, "cores": 1, "kind": "oracle", "core": core,
             "sample": f"{done} rows of the timed lists (memcpy per row, {t_total:.1f} s single-threaded C)",
             "host_cores": os.cpu_count(), "ranks": d.world}, parity)


# ----------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ----------------------------------------------------------------------------------------------
def run_reference(args, d: Dist):
    import oracle
    if d.rank != 0:
        return None
    K, W = args.steps, args.warmup
    # one core of GPU 0's NUMA node (any allowed core without a GPU)
    core = rank_cpu_share(_SoloDist())[0][0] if torch.cuda.is_available() else sorted(os.sched_getaffinity(0))[0]
    os.sched_setaffinity(0, {core})
    common = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": d.world, "steps": K, "warmup": W,
              "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "data": "synthetic", "gpu_launches": 0}
    if args.config == 5:
        c4 = sweep_buffer_cfg(args)
        R, base = args.row_bytes, args.base
        total = c4.table_bytes
        rows = (total - base) // R
        raw = np.empty(total + 4096, dtype=np.uint8)
        gen.fill_table(raw, total, c4.seed)
        n = min(rows, SWEEP_BYTES // R)
        nsub = max(1, n // 16)      # a bounded sample of each list (1/16), so the run ends in minutes
        want = np.empty(nsub * R, dtype=np.uint8)

        def one(i):
            ids = sweep_ids(rows, n, 0, i, R, base)[:nsub]
            oracle.gather_into(raw.ctypes.data + base, rows, R, ids, want)
            return nsub
        for i in range(W):
            one(i)
        t0 = time.perf_counter()
        tot = sum(one(i) for i in range(W, W + K))
        el = time.perf_counter() - t0
        value = tot * R / el / 1e9
        sample = f"{K} steps, each the first 1/16 ({nsub} rows) of that step's list (memcpy per row, single-threaded C)"
        dt = f"u8 ({args.dtype} rows moved as bytes)"
    else:
        cfg = gen.CONFIGS[args.config]
        R = cfg.row_bytes
        nbytes = cfg.table_bytes
        raw = np.empty(nbytes + 64, dtype=np.uint8)
        gen.fill_table(raw, nbytes, cfg.seed)
        off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed,
                               skew_alpha=args.skew_alpha if args.cache_frac > 0 else 0.0)
        out = np.empty(gen.sample_bound(cfg.n_nodes, cfg.batch, cfg.fanouts)[-1] * R, dtype=np.uint8)

        def one(j):
            seeds = gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j)
            s, _ = oracle.sample_and_gather(off, col, seeds, cfg.fanouts, gen.batch_rng_seed(cfg.seed, j), raw.ctypes.data,
                                            cfg.n_nodes, R, out=out)
            return s.U.shape[0]
        for i in range(W):
            one(i)
        t0 = time.perf_counter()
        tot = sum(one(i) for i in range(W, W + K))
        el = time.perf_counter() - t0
        value = tot * R / el / 1e9
        sample = f"{K} config{cfg.cid} minibatches, one per step (sample + gather, single-threaded C)"
        dt = "u8 (fp32 rows moved as bytes)"
    return dict(common, value=round(value, 4), ms_per_step=round(el / K * 1e3, 3), dtype=dt,
                config={"workload": workload_name(args), "parallelism": "cpu (rank 0 only)"},
                cpu_baseline={"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle", "core": core,
                              "sample": sample},
                e2e={"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})


class _SoloDist:
    """A one-rank stand-in for Dist (the reference arm runs on rank 0 alone)."""
    world, rank, pg = 1, 0, None

    def gather_obj(self, obj):
        return [obj]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--row-bytes", type=int, default=512, help="config 5: row width in bytes")
    ap.add_argument("--base", type=int, default=0, help="config 5: byte offset of row 0 in the host buffer")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16"], help="config 5: element type of the rows")
    ap.add_argument("--table-gb", type=float, default=0.0,
                    help="config 5: host buffer size in GB (default 0 = the config-4 table, 56.9 GB; tests shrink it)")
    ap.add_argument("--cache-frac", type=float, default=0.0,
                    help="configs 1-4: cache this fraction of the rows (highest in-degree) in HBM, sharded over the ranks "
                         "(NEXT-1), on the power-law variant of the graph")
    ap.add_argument("--skew-alpha", type=float, default=3.0, help="power-law exponent of the graph with --cache-frac")
    ap.add_argument("--host-table", default="auto", choices=["auto", "managed", "registered"],
                    help="feature table in managed host memory (large GPU pages) or cudaHostRegister'd (the paper's "
                         "unified tensor, one shared copy per box); auto: managed when every rank can hold a copy")
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
                    help="warps per SM of every overlap candidate (0: each candidate's own)")
    ap.add_argument("--consumer", default="sage", choices=["sage", "mean"],
                    help="overlap leg's stand-in consumer: the GraphSAGE layer (mean + GEMM, a7) or the mean alone")
    ap.add_argument("--consumer-hidden", type=int, default=256, help="the layer's output width (a multiple of 16, <= 256)")
    ap.add_argument("--overlap-slots", type=int, default=2,
                    help="overlap leg: minibatch buffers in the ring (2 = ping-pong, P:546-561; 3 fetches two ahead)")
    ap.add_argument("--consumer-ctas-per-sm", type=int, default=0,
                    help="the layer as one persistent launch of this many CTAs per SM per step (0: `repeat` short launches)")
    ap.add_argument("--timeline", default=None, help="write the overlap leg's best-shape timeline as a Chrome trace here")
    ap.add_argument("--oracle-budget", type=float, default=20.0, help="seconds of oracle work in the cpu_baseline leg")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--no-overlap", dest="overlap", action="store_false")
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"
    d = Dist(args.gpus)
    try:
        if args.impl == "reference":
            line = run_reference(args, d)
        elif args.config == 5:
            line = run_rowsweep(args, d)
        else:
            line = run_ours(args, d)
        if d.rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    except PreflightError as e:
        if d.rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": d.world,
                              "error": f"preflight: {e}"}), flush=True)
        sys.exit(3)
    finally:
        d.close()


if __name__ == "__main__":
    main()
