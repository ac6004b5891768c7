"""GraphSAGE minibatch training fed three ways (the fig:eval_overall analogue).

The paper's application: DGL GraphSAGE training whose node features live in host
memory.  Strategies compared on the same minibatches (GPU sampler, same model, same optimizer):

  zc   -- this repo's path: the fetch (sampler + address-sorted zero-copy gather, MinibatchFetcher)
          runs on a small green-context SM partition while training runs on the rest; step j+1 is
          fetched while step j trains (MPS X% / (100-X)% in the paper);
  dma  -- the paper's baseline: the sampled IDs go to the host, CPU threads gather the
          rows into pinned staging (torch.index_select), cudaMemcpyAsync H2D; double-buffered so the
          CPU gather of j+1 overlaps the training of j;
  hbm  -- "All-in-GPU": the whole table copied into HBM once (56.9 GB fits B200's
          180 GB) and gathered by the same kernel at HBM speed -- the lower bound on step time;
  uvm / uvm_host -- the UVM strategy: the table in CUDA managed memory, migrated into HBM
          on GPU page faults (uvm; the first pass is the cold cost) or kept in host memory and read
          through the GPU's mapping (uvm_host: preferred location CPU, accessed by the GPU).

The model is plain PyTorch (mean-aggregator SAGE layers): it is not the hot path, the
fetch is.  The table holds random bytes, not meaningful features: inputs are clamped to finite
values, labels are synthetic (seed ID mod classes).

    python examples/graphsage_train.py [--config 4] [--steps 20] [--modes zc,dma,hbm] [--fetch-sms 32] [--fetch-warps 2] [--contiguous] [--tune]
    torchrun --nproc-per-node N examples/graphsage_train.py --modes zc,dma     (DDP, one process per GPU)

Prints one JSON line: per mode the pipelined step time, the training time alone, and speedups.
"""
import argparse
import json
import os
import queue
import sys
import threading
import time

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import dgz_inputs as gen  # noqa: E402
from paper_2103_03330_b200 import dgz  # noqa: E402
from paper_2103_03330_b200.pipeline import MinibatchFetcher  # noqa: E402


class SAGE(torch.nn.Module):
    """L mean-aggregator SAGE layers: h'_v = act(W_self h_v + W_nbr mean_{u in S(v)} h_u)."""

    def __init__(self, d_in, hidden, classes, layers):
        super().__init__()
        dims = [d_in] + [hidden] * (layers - 1) + [classes]
        self.self_lin = torch.nn.ModuleList(torch.nn.Linear(dims[i], dims[i + 1]) for i in range(layers))
        self.nbr_lin = torch.nn.ModuleList(torch.nn.Linear(dims[i], dims[i + 1], bias=False) for i in range(layers))

    def forward(self, x, blocks, sizes):
        # blocks[k] = (positions in U [n_k, f_k] (-1 padded), counts [n_k]); the outermost hop first
        h = x
        L = len(blocks)
        for i, k in enumerate(reversed(range(L))):
            loc, cnt = blocks[k]
            n_dst = sizes[k]
            mask = (loc >= 0).unsqueeze(-1).to(h.dtype)
            nb = h[loc.clamp(min=0).long()] * mask                      # [n_dst, f, d]
            mean = nb.sum(1) / cnt.clamp(min=1).unsqueeze(-1).to(h.dtype)
            h = self.self_lin[i](h[:n_dst]) + self.nbr_lin[i](mean)
            if i < L - 1:
                h = F.relu(h)
        return h


class Trainer:
    def __init__(self, c, hidden, classes, ddp: bool = False):
        self.c = c
        self.classes = classes
        torch.manual_seed(0)
        self.model = SAGE(c.dim, hidden, classes, len(c.fanouts)).cuda()
        if ddp:   # data parallel over the ranks: gradients all-reduced by DDP (not the fetch path)
            self.model = torch.nn.parallel.DistributedDataParallel(self.model, device_ids=[torch.cuda.current_device()])
        self.opt = torch.optim.Adam(self.model.parameters(), lr=1e-3)

    def step(self, rows, bufs, sizes):
        c = self.c
        n = sizes[-1]
        x = torch.nan_to_num(rows[:n].view(torch.float32).view(n, c.dim), nan=0.0, posinf=1.0, neginf=-1.0)
        x = x.clamp(-1e3, 1e3)
        labels = (bufs.ids[:sizes[0]] % self.classes).long()        # synthetic labels of the seeds
        blocks = [(loc, cnt) for (nbr, cnt, loc) in bufs.hop_blocks(sizes)]
        out = self.model(x, blocks, sizes)
        loss = F.cross_entropy(out, labels)
        self.opt.zero_grad(set_to_none=True)
        loss.backward()
        self.opt.step()
        return loss


def timed(fn, K):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3 / K, r


def dump_minibatch(path, j, ids, rows, blocks=None):
    """Write one fetched minibatch (global batch j: U, its rows, per-hop counts / positions in U) to an
    .npz file, so that a test can check what the training consumed against the CPU oracle."""
    d = {"j": np.int64(j), "U": ids.cpu().numpy(), "rows": rows.cpu().numpy()}
    for k, (cnt, loc) in enumerate(blocks or []):
        d[f"cnt{k}"] = cnt.cpu().numpy()
        d[f"loc{k}"] = loc.cpu().numpy()
    np.savez(path, **d)


def run_fetcher_mode(table, graph, c, seeds, rng, K, fetch_sms, make_trainer, sample_on="compute", spread=False,
                     tune=False, fetch_warps=8, dump=None, order=None, cold=False):
    """zc / hbm: gather on a `fetch_sms` green-context partition, training on the others.  The
    sampler (HBM-bound, ~0.3 ms on the big partition) runs either in the training stream between
    steps (`compute`) or in front of the gather on the fetch partition (`fetch`)."""
    tuned = None
    if tune:   # time a few partition shapes UNDER training load on this chip and keep the fastest
        from paper_2103_03330_b200.pipeline import tune_fetch_partition
        probe = make_trainer()          # a throw-away model: the consumer the candidates are timed beside

        def consumer(mb, stream):
            sz = mb.sizes()
            with torch.cuda.stream(stream):
                probe.step(mb.rows, mb.bufs, sz)
        cands = [{"sms": k, "flags": dgz.PARTITION_SPREAD, "warps": w} for k, w in ((16, 3), (24, 2), (32, 2), (32, 3), (24, 8))]
        part, pcfg, tuned = tune_fetch_partition(table, graph, c.fanouts, c.batch, seeds[:6], rng[:6], candidates=cands,
                                                 consumer=consumer)
        del probe
    else:
        part = dgz.Partition(fetch_sms, -1, dgz.PARTITION_SPREAD if spread else 0)
        pcfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=fetch_warps,
                              flags=dgz.FLAG_DEEP | (0 if os.environ.get("DGZ_TRAIN_STATIC") == "1" else dgz.FLAG_DYNAMIC))
    comp = part.compute_stream
    f = MinibatchFetcher(table, graph, c.fanouts, c.batch, fetch_stream=part.fetch_stream, gather_cfg=pcfg,
                         sample_stream=comp if sample_on == "compute" else None, order=order)
    with torch.cuda.stream(comp):   # model (and DDP's buckets) created on the stream that trains
        trainer = make_trainer()
    torch.cuda.synchronize()

    def fetch_alone():
        for i in range(K):
            f.fetch(seeds[i], rng[i]).sizes()
    t_first = timed(fetch_alone, K)[0] if cold else None   # the first pass over a cold table (UVM: page faults)
    for i in range(2):
        fetch_alone()
    t_fetch, _ = timed(fetch_alone, K)
    mb = f.fetch(seeds[0], rng[0])
    sz = mb.sizes()
    if dump:   # (path, j): the minibatch every timed loop starts with, as the model sees it
        n = sz[-1]
        dump_minibatch(dump[0], dump[1], mb.bufs.ids[:n], mb.rows[:n],
                       [(cnt, loc) for (nbr, cnt, loc) in mb.bufs.hop_blocks(sz)])
    with torch.cuda.stream(comp):
        for _ in range(2):
            trainer.step(mb.rows, mb.bufs, sz)
        t_train, _ = timed(lambda: [trainer.step(mb.rows, mb.bufs, sz) for _ in range(K)], K)
    f.release(mb, comp)

    def pipelined():
        loss = None
        cur = f.fetch(seeds[0], rng[0])
        for i in range(1, K + 1):
            nxt = f.fetch(seeds[i], rng[i])     # fetch j+1 on the fetch partition ...
            s = cur.sizes()                      # (the host needs |F_k| to slice the blocks)
            with torch.cuda.stream(comp):
                comp.wait_event(cur.event)
                loss = trainer.step(cur.rows, cur.bufs, s)   # ... while j trains on the rest
            f.release(cur, comp)
            cur = nxt
        return loss.detach()
    pipelined()
    t_pipe, loss = timed(pipelined, K)
    out = {"step_ms": round(t_pipe, 3), "fetch_alone_ms": round(t_fetch, 3), "train_alone_ms": round(t_train, 3),
           "exposed_fetch_ms": round(max(0.0, t_pipe - t_train), 3), "loss": round(float(loss), 4),
           "fetch_sms": part.fetch_sms, "train_sms": part.compute_sms, "sampler_on": sample_on,
           "fetch_partition": ("tuned: " + json.dumps(tuned)) if tuned else ("spread over the GPCs" if spread else "contiguous"),
           "fetch_warps_per_sm": pcfg.warps_per_cta,
           "rows_per_minibatch": sz[-1]}
    if t_first is not None:
        out["first_pass_fetch_ms"] = round(t_first, 3)
    f.close()
    torch.cuda.synchronize()
    part.destroy()
    return out


def managed_table(c, buf, host_preferred):
    """The UVM strategy: the table in CUDA managed memory, filled by the CPU (so it starts
    resident in host memory).  host_preferred=False: the default policy -- GPU accesses fault and the
    driver migrates pages into HBM (B200's HBM holds the whole table, so later passes run from HBM);
    True: cudaMemAdviseSetPreferredLocation(CPU) + SetAccessedBy(GPU) -- pages stay in host memory and
    the GPU reads them through its mapping (UVM's own zero-copy).  Returns (pointer, free())."""
    import ctypes
    from cuda.bindings import runtime as rt
    err, ptr = rt.cudaMallocManaged(c.table_bytes, rt.cudaMemAttachGlobal)
    assert err == rt.cudaError_t.cudaSuccess, err
    dst = np.ctypeslib.as_array((ctypes.c_uint8 * c.table_bytes).from_address(int(ptr)))
    src = buf.numpy(0, c.table_bytes)
    step = 1 << 30
    for o in range(0, c.table_bytes, step):
        dst[o:o + step] = src[o:o + step]
    if host_preferred:
        dev = torch.cuda.current_device()
        for adv, where in ((rt.cudaMemoryAdvise.cudaMemAdviseSetPreferredLocation, rt.cudaCpuDeviceId),
                           (rt.cudaMemoryAdvise.cudaMemAdviseSetAccessedBy, dev)):
            (e,) = rt.cudaMemAdvise(ptr, c.table_bytes, adv, where)
            assert e == rt.cudaError_t.cudaSuccess, e
    return int(ptr), (lambda: rt.cudaFree(ptr))


def run_dma_mode(host_rows, graph, c, seeds, rng, K, threads, trainer, dump=None):
    """The paper's DMA-based method, pipelined: a worker thread samples on the GPU,
    copies U to the host, gathers the rows with `threads` CPU threads into pinned staging and
    copies them H2D; the main thread trains on the previous minibatch meanwhile."""
    torch.set_num_threads(threads)
    R = c.row_bytes
    L = len(c.fanouts)
    bufs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts, blocks=True, local=True) for _ in range(2)]
    cap = bufs[0].bounds[-1]
    stage = [torch.empty((cap, R), dtype=torch.uint8).pin_memory() for _ in range(2)]
    ids_h = [torch.empty(cap, dtype=torch.int64).pin_memory() for _ in range(2)]
    rows = [torch.empty((cap, R), dtype=torch.uint8, device="cuda") for _ in range(2)]
    s_fetch = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for e in free:
        e.record()
    t_cpu = []

    def produce(q, slots, lo, hi):
        for i in range(lo, hi):
            p = slots.get()                             # the main thread has enqueued slot p's last training step
            assert p == i % 2
            free[p].synchronize()                       # ... and that step has finished on the GPU
            b = bufs[p]
            with torch.cuda.stream(s_fetch):
                dgz.sample_uniform(graph, seeds[i], c.fanouts, rng[i], b, stream=s_fetch)
                s_fetch.synchronize()
                n = int(b.sizes_host[-1])
                ids_h[p][:n].copy_(b.ids[:n])            # D2H of the sampled ID list
                t0 = time.perf_counter()
                torch.index_select(host_rows, 0, ids_h[p][:n], out=stage[p][:n])   # CPU gather
                t_cpu.append(time.perf_counter() - t0)
                rows[p][:n].copy_(stage[p][:n], non_blocking=True)                # H2D DMA
                ready[p].record(s_fetch)
            q.put((p, b.sizes_host.tolist()))
        q.put(None)

    def loop(lo, hi):
        q = queue.Queue(maxsize=1)
        slots = queue.Queue()                           # slot tokens: a slot is re-filled only after its
        slots.put(lo % 2)                               # training step was enqueued (free[p] recorded)
        slots.put((lo + 1) % 2)
        th = threading.Thread(target=produce, args=(q, slots, lo, hi), daemon=True)
        th.start()
        loss = None
        while True:
            item = q.get()
            if item is None:
                break
            p, sz = item
            cur = torch.cuda.current_stream()
            cur.wait_event(ready[p])
            loss = trainer.step(rows[p], bufs[p], sz)
            free[p].record(cur)
            slots.put(p)
        th.join()
        return loss.detach()
    loop(0, 2)
    t_cpu.clear()

    def fetch_alone():
        for i in range(K):
            p = i % 2
            b = bufs[p]
            dgz.sample_uniform(graph, seeds[i], c.fanouts, rng[i], b, stream=s_fetch)
            s_fetch.synchronize()
            n = int(b.sizes_host[-1])
            ids_h[p][:n].copy_(b.ids[:n])
            torch.index_select(host_rows, 0, ids_h[p][:n], out=stage[p][:n])
            with torch.cuda.stream(s_fetch):
                rows[p][:n].copy_(stage[p][:n], non_blocking=True)
        s_fetch.synchronize()
    t_fetch, _ = timed(fetch_alone, K)
    if dump:   # the last minibatch fetch_alone staged: slot (K-1) % 2, global batch dump[1]
        p = (K - 1) % 2
        n = int(bufs[p].sizes_host[-1])
        dump_minibatch(dump[0], dump[1], ids_h[p][:n], rows[p][:n])
    t_pipe, loss = timed(lambda: loop(0, K), K)
    return {"step_ms": round(t_pipe, 3), "fetch_alone_ms": round(t_fetch, 3), "cpu_gather_ms": round(1e3 * float(np.median(t_cpu)), 3),
            "cpu_threads": threads, "loss": round(float(loss), 4)}


def load_graph(c, G, rank, dist):
    """The CSR in this GPU's HBM.  With G > 1 ranks rank 0 generates it once into /dev/shm and every
    rank maps it (one host copy per box, as for the table) before uploading its own HBM copy."""
    if G == 1:
        off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
        return dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    base = f"/dgz_train_csr_{os.environ.get('MASTER_PORT', '0')}"
    bufs = []
    e = [None]
    if rank == 0:
        def alloc(nb):
            b = dgz.HostBuffer(nb + 4096, shm_name=f"{base}_{len(bufs)}", create=True)
            bufs.append(b)
            return b.ptr
        _, _, e[0] = gen.gen_csr_into(c.n_nodes, c.avg_degree, c.seed, alloc)
    dist.broadcast_object_list(e, src=0)
    if rank != 0:
        for i, nb in enumerate(((c.n_nodes + 1) * 8, max(e[0] * 4, 1))):
            bufs.append(dgz.HostBuffer(nb + 4096, shm_name=f"{base}_{i}", create=False))
    dist.barrier()
    off = torch.from_numpy(bufs[0].numpy(0, (c.n_nodes + 1) * 8).view(np.int64)).cuda()
    col = torch.from_numpy(bufs[1].numpy(0, e[0] * 4).view(np.int32)).cuda()
    dist.barrier()
    if rank == 0:
        for b in bufs:
            b.unlink()
    for b in bufs:
        b.free()
    return dgz.Graph(off, col)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--dim", type=int, default=0, help="override the feature dimension (fig:eval_sweep analogue)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--hidden", type=int, default=256)
    ap.add_argument("--classes", type=int, default=172)      # ogbn-papers100M has 172 classes
    ap.add_argument("--modes", default="zc,dma,hbm", help="any of zc, dma, hbm, uvm, uvm_host")
    ap.add_argument("--fetch-sms", type=int, default=32)
    ap.add_argument("--sample-on", default="compute", choices=["compute", "fetch"])
    ap.add_argument("--contiguous", dest="spread", action="store_false",
                    help="fetch SMs contiguous in the split (default: spread over the GPCs)")
    ap.add_argument("--tune", action="store_true", help="time a few fetch partitions first and keep the fastest")
    ap.add_argument("--fetch-warps", type=int, default=2,
                    help="warps per SM of the partition's gather (few: beside training the page walks slow down)")
    ap.add_argument("--threads", type=int, default=max(1, (os.cpu_count() or 2) - 1))   # one core left for the training loop
    ap.add_argument("--host-table", default="registered", choices=["registered", "managed"],
                    help="zc mode's host table: cudaHostRegister'd (the paper's) or DGZ_HOST_MANAGED")
    ap.add_argument("--dump", default=None,
                    help="directory: write the first zc minibatch and the last DMA minibatch of each rank as .npz")
    a = ap.parse_args()
    # one process per GPU under torchrun (DDP; DGZ_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 with gloo)
    G = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    same = os.environ.get("DGZ_BENCH_SAME_DEVICE") == "1"
    dev_id = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev_id)
    dist = None
    if G > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if same else "nccl")
    torch.backends.cuda.matmul.allow_tf32 = True
    c = gen.CONFIGS[a.config]
    if a.dim:
        import dataclasses
        c = dataclasses.replace(c, dim=a.dim)
    K = a.steps
    if a.host_table == "managed":   # one DGZ_HOST_MANAGED copy per rank (2 MiB GPU pages)
        buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_MANAGED)
        gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    elif G == 1:
        buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
        gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    else:   # one host table per box, registered by every rank
        name = f"/dgz_train_{os.environ.get('MASTER_PORT', '0')}"
        if rank == 0:
            buf = dgz.HostBuffer(c.table_bytes + 4096, shm_name=name, create=True)
            gen.fill_table(buf.ptr, c.table_bytes, c.seed)
        dist.barrier()
        if rank != 0:
            buf = dgz.HostBuffer(c.table_bytes + 4096, shm_name=name, create=False)
        dist.barrier()
        if rank == 0:
            buf.unlink()
    table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    graph = load_graph(c, G, rank, dist)
    batches = [i * G + rank for i in range(K + 2)]          # seed partition: global batch j = i*G + rank
    seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in batches]
    rng = [gen.batch_rng_seed(c.seed, j) for j in batches]
    res = {"config": c.name, "dim": c.dim, "steps": K, "ranks": G, "host_table": a.host_table, "model": f"GraphSAGE-mean {len(c.fanouts)} layers, hidden {a.hidden}, "
                                                              f"{a.classes} classes, Adam, fp32 (TF32 matmuls)"
                                                              + (", DDP" if G > 1 else "")}
    modes = a.modes.split(",")
    threads = max(1, a.threads // G)
    if a.dump:
        os.makedirs(a.dump, exist_ok=True)
    if "zc" in modes:
        res["zc"] = run_fetcher_mode(table, graph, c, seeds, rng, K, a.fetch_sms,
                                     lambda: Trainer(c, a.hidden, a.classes, G > 1), a.sample_on, a.spread, a.tune,
                                     a.fetch_warps,
                                     dump=(os.path.join(a.dump, f"zc_rank{rank}.npz"), batches[0]) if a.dump else None)
    if "dma" in modes:
        host_rows = torch.from_numpy(buf.numpy(0, c.table_bytes)).view(c.n_nodes, c.row_bytes)
        res["dma"] = run_dma_mode(host_rows, graph, c, seeds, rng, K, threads, Trainer(c, a.hidden, a.classes, G > 1),
                                  dump=(os.path.join(a.dump, f"dma_rank{rank}.npz"), batches[K - 1]) if a.dump else None)
    if "hbm" in modes:
        dev = torch.empty(c.table_bytes, dtype=torch.uint8, device="cuda")
        dev.copy_(torch.from_numpy(buf.numpy(0, c.table_bytes)))
        dtab = dgz.DeviceTable(dev.data_ptr(), c.n_nodes, c.dim, dgz.F32)
        res["hbm"] = run_fetcher_mode(dtab, graph, c, seeds, rng, K, a.fetch_sms,
                                      lambda: Trainer(c, a.hidden, a.classes, G > 1), a.sample_on, a.spread, a.tune,
                                     a.fetch_warps)
        dtab.unregister()
        del dev
    for m in ("uvm", "uvm_host"):   # the paper's UVM strategy, both placements (same fetcher, address order)
        if m in modes:
            ptr, free = managed_table(c, buf, host_preferred=(m == "uvm_host"))
            utab = dgz.DeviceTable(ptr, c.n_nodes, c.dim, dgz.F32)
            res[m] = run_fetcher_mode(utab, graph, c, seeds, rng, K, a.fetch_sms,
                                      lambda: Trainer(c, a.hidden, a.classes, G > 1), a.sample_on, a.spread, a.tune,
                                      a.fetch_warps, order="sorted", cold=True)
            utab.unregister()
            torch.cuda.synchronize()
            free()
    if G > 1:   # per-rank results to rank 0; the job's step time is the slowest rank's
        allres = [None] * G
        dist.all_gather_object(allres, {m: res[m] for m in ("zc", "dma", "hbm", "uvm", "uvm_host") if m in res})
        for m in ("zc", "dma", "hbm", "uvm", "uvm_host"):
            if m in res:
                res[m] = {"step_ms": max(r[m]["step_ms"] for r in allres), "per_rank": [r[m] for r in allres]}
    if "zc" in res and "dma" in res:
        res["speedup_zc_over_dma"] = round(res["dma"]["step_ms"] / res["zc"]["step_ms"], 3)
    if "zc" in res and "hbm" in res:
        res["zc_vs_all_in_gpu"] = round(res["hbm"]["step_ms"] / res["zc"]["step_ms"], 3)
    for m in ("uvm", "uvm_host"):
        if "zc" in res and m in res:
            res[f"speedup_zc_over_{m}"] = round(res[m]["step_ms"] / res["zc"]["step_ms"], 3)
    if rank == 0:
        print(json.dumps(res), flush=True)
    table.unregister()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()
    buf.free()


if __name__ == "__main__":
    main()
