"""Per-GPU minibatch fetch pipeline (steps a2-a5): sampler -> zero-copy gather into ping-pong
HBM buffers on a side stream, consumed on another stream (section 3.3,
fig:singlegpu; section 3.2.2).

The paper runs sampler, producer (gather) and consumer (training) as three processes and
shares the ping-pong buffers with CUDA IPC, limiting the producer to X% of the SMs with MPS.
On B200 one process per GPU does it with two CUDA streams and events: the fetch for step j+1
is enqueued on ``fetch_stream`` into the other slot while the consumer works on slot j, the
gather's grid is bounded to a few SMs (``gather_cfg.sm_count``), nothing allocates or blocks
inside the loop, and the whole fetch (sampling + gather) runs on the device with
the data-dependent sizes kept in device memory.  Everything compute-related is a libdgz call.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import dgz


@dataclass
class Minibatch:
    slot: int
    bufs: dgz.SampleBuffers
    rows: torch.Tensor          # [cap, row_bytes] uint8 in HBM: row r = table[ids[r]]
    event: torch.cuda.Event     # recorded on the gather stream after the gather
    fanouts: tuple
    timing: tuple | None = None  # (sample start, gather start, gather end) timing events

    @property
    def n_dev(self) -> torch.Tensor:
        L = len(self.fanouts)
        return self.bufs.sizes_dev[L:L + 1]

    def wait(self, stream=None) -> None:
        (torch.cuda.current_stream() if stream is None else stream).wait_event(self.event)

    def sizes(self) -> list:
        """|F_0..F_L| (synchronises with the fetch)."""
        self.event.synchronize()
        return self.bufs.sizes_host.tolist()


class MinibatchFetcher:
    """Owns ping-pong sample buffers and row buffers for one GPU and one registered table.

    Default (``sampler_sms=8``): the device is split with green contexts (``dgz.Partition``)
    into a small sampler group and a gather group, and the sampler of minibatch j+1 runs on its
    8 SMs while minibatch j is gathered on the others -- the ~0.3 ms of sampling disappears from
    the step (measured: 49.5 vs 46.6 GB/s).  Sampling on a second stream over the WHOLE GPU is
    much worse (27 GB/s: its full-GPU bitmap passes stall the translation-bound gather), so
    without green contexts (``sampler_sms=0``) both phases run back to back on one high-priority
    stream.  Slot reuse is ordered by events either way (a slot is resampled only after its gather
    and its consumer are done).  An explicit ``fetch_stream`` (e.g. a partition shared with a
    consumer) is used for both phases unless ``sample_stream`` is given too.
    """

    def __init__(self, table: dgz.Table, graph: dgz.Graph, fanouts, max_seeds: int, slots: int = 2,
                 gather_cfg: dgz.GatherCfg | None = None, blocks: bool = True, fetch_stream=None,
                 overlap_sampling: bool = False, sample_stream=None, sampler_sms: int | None = None, graphs: bool = False,
                 cache=None, order: str | None = None):
        self.table, self.graph = table, graph
        # an HBM hot-row cache (dgz.HotRowCache / dgz.ShardedHotRowCache, NEXT-1): the gather reads
        # cached rows from HBM (this GPU's or a peer's shard) and only the rest over PCIe
        self.cache = cache
        # an HBM-resident table (dgz.DeviceTable) is gathered in frontier order (explore31)
        self.hbm_table = bool(table.info.flags & dgz.REG_DEVICE)
        if order is not None:      # "sorted" (address order) / "frontier": override the table-kind default
            assert order in ("sorted", "frontier")
            self.hbm_table = order == "frontier"
        if sampler_sms is None:
            # A zero-copy CSR (dgz.HostGraph) makes the sampler a stream of small PCIe reads: beside
            # the gather both slow down (36 vs 37.8 GB/s sequential, config 4), so it runs back to
            # back with the gather on the whole GPU; an HBM CSR samples on 8 SMs, hidden.
            sampler_sms = 0 if isinstance(graph, dgz.HostGraph) else 8
        self.fanouts = tuple(int(f) for f in fanouts)
        self.max_seeds = max_seeds
        self.cfg = gather_cfg
        # high priority: the fetch's few CTAs are scheduled ahead of the consumer's as SMs free up
        self.partition = None
        self.mode = "sequential"
        self.graphs = graphs
        if graphs:                        # one CUDA graph per slot on ordinary streams
            sampler_sms = 0
            overlap_sampling = False
        if fetch_stream is None and sample_stream is None and sampler_sms > 0 and not overlap_sampling:
            try:
                self.partition = dgz.Partition(sampler_sms, -1, dgz.PARTITION_SPREAD)
            except dgz.DgzError:
                self.partition = None      # no green contexts: sequential scheduling below
        if self.partition is not None:
            self.sample_stream = self.partition.fetch_stream
            self.stream = self.partition.compute_stream
            self.mode = f"sampler on {self.partition.fetch_sms} SMs | gather on {self.partition.compute_sms} SMs"
        elif fetch_stream is None:
            self.stream = torch.cuda.Stream(priority=-1)
            self.sample_stream = torch.cuda.Stream(priority=-1) if overlap_sampling else self.stream
            if overlap_sampling:
                self.mode = "sampler and gather on two full-GPU streams"
        else:
            self.stream = self.sample_stream = fetch_stream
        if sample_stream is not None:          # e.g. a small green-context partition for the sampler
            self.sample_stream = sample_stream
            self.mode = "caller-provided sampler stream"
        self.bufs = [dgz.SampleBuffers(graph.n_nodes, max_seeds, self.fanouts, blocks=blocks, local=blocks,
                                       sorted_ids=True, device_rng=graphs) for _ in range(slots)]
        self.cuda_graphs = [None] * slots
        self.graph_kernels = 0     # libdgz kernels per graph replay (counted at capture)
        self.graph_replays = 0
        if graphs:
            self.mode = "sequential, one CUDA graph per slot (sampler + gather replayed as one launch)"
        cap = self.bufs[0].bounds[-1]
        self.rows = [torch.empty((cap, table.row_bytes), dtype=torch.uint8, device="cuda") for _ in range(slots)]
        self.seed_stage = [torch.empty(max_seeds, dtype=torch.int64, device="cuda") for _ in range(slots)]
        self.events = [torch.cuda.Event() for _ in range(slots)]      # gather of slot p done
        self.sampled = [torch.cuda.Event() for _ in range(slots)]     # sampling of slot p done
        self.free = [torch.cuda.Event() for _ in range(slots)]        # consumer of slot p done
        self.next_slot = 0

    def close(self) -> None:
        """Destroy the green-context partition (after all queued work finished)."""
        if self.partition is not None:
            torch.cuda.synchronize()
            self.partition.destroy()
            self.partition = None

    def release(self, mb: Minibatch, stream=None) -> None:
        """Mark slot `mb.slot` reusable once the consumer's queued work on `stream` is done."""
        self.free[mb.slot].record(torch.cuda.current_stream() if stream is None else stream)

    def fetch(self, seeds: torch.Tensor, rng_seed: int, slot: int | None = None, timing: bool = False,
              count_into: torch.Tensor | None = None) -> Minibatch:
        """Enqueue sampling + gather of one minibatch (seeds: int64, on the device or pinned host; a
        host tensor is copied asynchronously, so keep it unchanged until the minibatch's event).
        ``count_into``: a 1-element device int64 tensor that receives |U| on the gather stream."""
        p = self.next_slot if slot is None else slot
        self.next_slot = (p + 1) % len(self.bufs)
        ss, gs = self.sample_stream, self.stream
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
              torch.cuda.Event(enable_timing=True)) if timing else None
        # slot p's sampler outputs and rows are free once its previous gather and consumer are done
        ss.wait_event(self.events[p])
        ss.wait_event(self.free[p])
        n_seeds = seeds.numel()
        assert n_seeds <= self.max_seeds
        b = self.bufs[p]
        L = len(self.fanouts)
        if self.graphs and n_seeds == self.max_seeds:
            return self._fetch_graph(p, seeds, rng_seed, ev, count_into)
        torch.cuda.nvtx.range_push(f"dgz.sample slot {p}")   # host-side ranges for nsys timelines
        with torch.cuda.stream(ss):
            if ev:
                ev[0].record(ss)
            if not seeds.is_cuda:
                self.seed_stage[p][:n_seeds].copy_(seeds, non_blocking=True)   # H2D of the index list
                seeds = self.seed_stage[p][:n_seeds]
            if b.rng_dev is not None:
                b.rng_dev.fill_(_as_i64(rng_seed))
            dgz.sample_uniform(self.graph, seeds, self.fanouts, rng_seed, b, stream=ss)
            self.sampled[p].record(ss)
        torch.cuda.nvtx.range_pop()
        gs.wait_event(self.sampled[p])
        torch.cuda.nvtx.range_push(f"dgz.gather slot {p}")
        with torch.cuda.stream(gs):
            if ev:
                ev[1].record(gs)
            if self.hbm_table:   # All-in-GPU: no address translation to save; write rows in order
                dgz.gather(self.table, b.ids, self.rows[p], n=b.bounds[-1], n_dev=b.sizes_dev[L:L + 1],
                           cfg=self.cfg or dgz.gather_cfg(), stream=gs)
            elif self.cache is not None:
                self.cache.gather(b.ids_sorted, self.rows[p], dst_pos=b.ids_sorted_pos, n=b.bounds[-1],
                                  n_dev=b.sizes_dev[L:L + 1], cfg=self.cfg, stream=gs)
            else:
                dgz.gather_perm(self.table, b.ids_sorted, b.ids_sorted_pos, self.rows[p], n=b.bounds[-1],
                                n_dev=b.sizes_dev[L:L + 1], cfg=self.cfg, stream=gs)
            if ev:
                ev[2].record(gs)
            if count_into is not None:
                count_into.copy_(b.sizes_dev[L:L + 1], non_blocking=True)
            self.events[p].record(gs)
        torch.cuda.nvtx.range_pop()
        return Minibatch(p, b, self.rows[p], self.events[p], self.fanouts, ev)

    # ---- CUDA-graph mode ----------------------------------------------------------------------
    def _enqueue_graph_body(self, p):
        b = self.bufs[p]
        L = len(self.fanouts)
        dgz.sample_uniform(self.graph, self.seed_stage[p], self.fanouts, 0, b, stream=self.stream)
        if self.hbm_table:
            dgz.gather(self.table, b.ids, self.rows[p], n=b.bounds[-1], n_dev=b.sizes_dev[L:L + 1],
                       cfg=self.cfg or dgz.gather_cfg(), stream=self.stream)
        elif self.cache is not None:
            self.cache.gather(b.ids_sorted, self.rows[p], dst_pos=b.ids_sorted_pos, n=b.bounds[-1],
                              n_dev=b.sizes_dev[L:L + 1], cfg=self.cfg, stream=self.stream)
        else:
            dgz.gather_perm(self.table, b.ids_sorted, b.ids_sorted_pos, self.rows[p], n=b.bounds[-1],
                            n_dev=b.sizes_dev[L:L + 1], cfg=self.cfg, stream=self.stream)

    def _fetch_graph(self, p, seeds, rng_seed, ev, count_into):
        """Sampler + gather of slot p as one CUDA-graph replay: seeds and the sampler seed are
        written into the graph's fixed input buffers first (launch-bound small minibatches)."""
        s = self.stream
        b = self.bufs[p]
        L = len(self.fanouts)
        if self.cuda_graphs[p] is None:
            with torch.cuda.stream(s):                  # eager warm-up (allocates lazy state)
                self.seed_stage[p].copy_(seeds, non_blocking=True)
                self._enqueue_graph_body(p)
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            k0 = dgz.kernel_launches()
            with torch.cuda.graph(g, stream=s):
                self._enqueue_graph_body(p)
            self.graph_kernels = dgz.kernel_launches() - k0   # libdgz kernels captured per replay
            self.cuda_graphs[p] = g
        with torch.cuda.stream(s):
            if ev:
                ev[0].record(s)
            self.seed_stage[p].copy_(seeds, non_blocking=True)
            b.rng_dev.fill_(_as_i64(rng_seed))
            if ev:
                ev[1].record(s)
            self.cuda_graphs[p].replay()
            self.graph_replays += 1
            if ev:
                ev[2].record(s)
            if count_into is not None:
                count_into.copy_(b.sizes_dev[L:L + 1], non_blocking=True)
            self.sampled[p].record(s)
            self.events[p].record(s)
        return Minibatch(p, b, self.rows[p], self.events[p], self.fanouts, ev)


def _as_i64(x: int) -> int:
    """uint64 sampler seed -> the int64 with the same bits (torch tensors are signed)."""
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= (1 << 63) else x


def tune_fetch_partition(table: dgz.Table, graph, fanouts, max_seeds: int, seeds, rng_seeds, candidates=None,
                         warps_per_cta: int = 2, consumer=None):
    """Pick the green-context partition whose SMs gather fastest on THIS chip (DESIGN.md section 5:
    at a fixed SM count the zero-copy gather's rate depends strongly and reproducibly on which SMs
    walk the GPU page tables, and the best set differs between chips).  Samples the given minibatches
    once, then times the address-sorted gather of all of them on each candidate partition (alone)
    and returns (best dgz.Partition, its gather config, [(candidate, GB/s), ...]); the other
    partitions are destroyed.  candidates: list of dicts with either {"sms": k, "flags": f} or
    {"groups": [...]} (dgz_partition_create_groups), optionally with "warps"; default: 24 and 32 SMs,
    contiguous and spread, with 2 warps per SM (few rows in flight: the page walks are what the gather
    waits on).  With ``consumer(minibatch, stream)`` -- e.g. one training step enqueued on `stream` --
    each candidate is instead timed UNDER LOAD: the fetch of step j+1 on the partition while the
    consumer works on step j on the other SMs, which is the shape that matters in training (the
    consumer's DRAM traffic slows the gather's page walks).  Results are then
    ms per pipelined step (lower is better) instead of GB/s."""
    if candidates is None:
        candidates = [{"sms": 24, "flags": 0}, {"sms": 24, "flags": dgz.PARTITION_SPREAD},
                      {"sms": 32, "flags": 0}, {"sms": 32, "flags": dgz.PARTITION_SPREAD}]
    fanouts = tuple(int(f) for f in fanouts)
    L = len(fanouts)
    bufs = []
    for s, r in zip(seeds, rng_seeds):
        b = dgz.SampleBuffers(graph.n_nodes, max_seeds, fanouts, blocks=False, local=False)
        dgz.sample_uniform(graph, s, fanouts, r, b)
        bufs.append(b)
    torch.cuda.synchronize()
    nbytes = sum(int(b.sizes_host[-1]) for b in bufs) * table.row_bytes
    out = torch.empty(max(b.bounds[-1] for b in bufs) * table.row_bytes, dtype=torch.uint8, device="cuda")
    results, best = [], None
    for cand in candidates:
        part = dgz.Partition(cand.get("sms", 0), -1, cand.get("flags", 0), groups=cand.get("groups"))
        cfg = dgz.gather_cfg(sm_count=part.fetch_sms, warps_per_cta=cand.get("warps", warps_per_cta),
                             flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)
        if consumer is not None:
            ms = _ms_per_loaded_step(table, graph, fanouts, max_seeds, seeds, rng_seeds, part, cfg, consumer)
            results.append((dict(cand, fetch_sms=part.fetch_sms), round(ms, 3)))
            if best is None or ms < best[2]:
                if best is not None:
                    best[0].destroy()
                best = (part, cfg, ms)
            else:
                part.destroy()
            continue
        s = part.fetch_stream
        b0 = bufs[0]
        dgz.gather_perm(table, b0.ids_sorted, b0.ids_sorted_pos, out, n=b0.bounds[-1], n_dev=b0.sizes_dev[L:L + 1],
                        cfg=cfg, stream=s)                       # warm-up
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for b in bufs:
            dgz.gather_perm(table, b.ids_sorted, b.ids_sorted_pos, out, n=b.bounds[-1], n_dev=b.sizes_dev[L:L + 1],
                            cfg=cfg, stream=s)
        e.record(s)
        e.synchronize()
        gbs = nbytes / (a.elapsed_time(e) * 1e-3) / 1e9
        results.append((dict(cand, fetch_sms=part.fetch_sms), round(gbs, 2)))
        if best is None or gbs > best[2]:
            if best is not None:
                best[0].destroy()
            best = (part, cfg, gbs)
        else:
            part.destroy()
    return best[0], best[1], results


def _ms_per_loaded_step(table, graph, fanouts, max_seeds, seeds, rng_seeds, part, cfg, consumer) -> float:
    """ms per pipelined step: fetch j+1 on the partition (sampler in the consumer's stream) while the
    consumer works on step j on the other SMs (second of two passes)."""
    import time
    f = MinibatchFetcher(table, graph, fanouts, max_seeds, fetch_stream=part.fetch_stream, gather_cfg=cfg,
                         sample_stream=part.compute_stream)
    comp = part.compute_stream
    out = 0.0
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cur = f.fetch(seeds[0], rng_seeds[0])
        for i in range(1, len(seeds) + 1):
            nxt = f.fetch(seeds[i], rng_seeds[i]) if i < len(seeds) else None
            comp.wait_event(cur.event)
            consumer(cur, comp)
            f.release(cur, comp)
            cur = nxt
        torch.cuda.synchronize()
        out = (time.perf_counter() - t0) * 1e3 / len(seeds)
    f.close()
    return out


def _ms_per_fetch(f: MinibatchFetcher, seeds, rng_seeds, reps: int = 2) -> float:
    """Steady-state ms per minibatch: from the end of the first gather to the end of the last (the
    pipeline's fill -- the first, unhidden sampling -- is not charged to either shape)."""
    assert len(seeds) >= 2
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f.fetch(seeds[0], rng_seeds[0])
        a.record(f.stream)
        for s, r in zip(seeds[1:], rng_seeds[1:]):
            f.fetch(s, r)
        b.record(f.stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / (len(seeds) - 1))
    return best


def calibrated_fetcher(table: dgz.Table, graph, fanouts, max_seeds: int, seeds, rng_seeds, **kw):
    """The default pipelined fetcher (sampler on an 8-SM green-context partition beside the gather) or
    the sequential one (sample, then gather, on the whole GPU), whichever fetches the given sample
    minibatches faster on THIS box: on most boxes the partitioned sampler is hidden for free, on some
    its memory traffic slows the gather's page walks by more than the ~0.3 ms it hides (DESIGN.md
    section 5).  Returns (fetcher, {"pipelined_ms_per_step", "sequential_ms_per_step", "chosen"});
    the losing fetcher is closed."""
    pipelined = MinibatchFetcher(table, graph, fanouts, max_seeds, **kw)
    if pipelined.partition is None:
        return pipelined, {"chosen": pipelined.mode, "note": "no green contexts: sequential only"}
    sequential = MinibatchFetcher(table, graph, fanouts, max_seeds, **dict(kw, sampler_sms=0))
    t_p = _ms_per_fetch(pipelined, seeds, rng_seeds)
    t_s = _ms_per_fetch(sequential, seeds, rng_seeds)
    keep, drop = (sequential, pipelined) if t_s < t_p else (pipelined, sequential)
    drop.close()
    return keep, {"pipelined_ms_per_step": round(t_p, 3), "sequential_ms_per_step": round(t_s, 3), "chosen": keep.mode}
