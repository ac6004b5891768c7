"""CUDA path (libdgz through its C ABI) vs the CPU oracle, element by element.

Bar: bit-exact (the gather moves bytes; the sampler is integer work).  Inputs come from
dgz_inputs; expected values come only from ``oracle``.
"""
import numpy as np
import pytest
import torch

import dgz_inputs as gen
import oracle

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2103_03330_b200 import dgz


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


class HostTable:
    """A host table at byte offset `base` inside a page-aligned mapping, registered."""

    def __init__(self, rows, row_bytes, seed, base=0, dtype=None, flags=0):
        dtype = dgz.U8 if dtype is None else dtype
        eb = dgz.ELEM_BYTES[dtype]
        assert row_bytes % eb == 0 and base % eb == 0
        self.rows, self.R, self.base = rows, row_bytes, base
        self.buf = dgz.HostBuffer(rows * row_bytes + base + 4096)
        arr = self.buf.numpy()
        gen.fill_table(arr.ctypes.data + base, rows * row_bytes, seed)
        self.np = arr[base:base + rows * row_bytes]
        self.table = dgz.register_table(self.buf.ptr + base, rows, row_bytes // eb, dtype, flags)

    def close(self):
        self.table.unregister()
        self.buf.free()


def _gather_dev(t, idx_np, cfg=None, out_offset=0, idx_dtype=torch.int64, n_dev=None, fill=0xAB):
    n = idx_np.shape[0]
    R = t.R
    raw = torch.full((n * R + 64,), fill, dtype=torch.uint8, device="cuda")
    out = raw[out_offset:out_offset + n * R]
    idx = torch.from_numpy(np.ascontiguousarray(idx_np)).to(device="cuda", dtype=idx_dtype)
    dgz.gather(t.table, idx, out, n=n, n_dev=n_dev, cfg=cfg)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(n, R) if n else np.zeros((0, R), np.uint8)


VARIANTS = [dgz.GATHER_SEGMENT, dgz.GATHER_BULK, dgz.GATHER_NAIVE, dgz.GATHER_SHIFT] if torch.cuda.is_available() else []


@pytest.mark.parametrize("R", gen.SWEEP_ROW_BYTES)
@pytest.mark.parametrize("base", gen.SWEEP_BASE_OFFSETS)
def test_gather_sweep_segment(dev, R, base):
    rows = max(64, min(4000, (8 << 20) // R))
    t = HostTable(rows, R, seed=R * 131 + base, base=base)
    try:
        idx = gen.random_ids(rows, 1000 + 17, seed=R + base)   # ragged tail (not a multiple of 32)
        want, bad = oracle.gather(t.np, R, idx)
        assert bad == 0
        got = _gather_dev(t, idx)
        assert np.array_equal(got, want)
    finally:
        t.close()


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
@pytest.mark.parametrize("R,base", [(512, 0), (400, 0), (2408, 0), (1028, 4), (100, 64), (16, 8), (4096, 16), (1044, 0)])
def test_gather_variants(dev, variant, R, base):
    rows = 3000
    t = HostTable(rows, R, seed=7 + R, base=base, dtype=dgz.F32)
    try:
        idx = gen.random_ids(rows, 777, seed=R)
        want, _ = oracle.gather(t.np, R, idx)
        for off in (0, 4, 8):
            got = _gather_dev(t, idx, cfg=dgz.gather_cfg(variant=variant), out_offset=off)
            assert np.array_equal(got, want), (variant, off)
    finally:
        t.close()


@pytest.mark.parametrize("dtype,dim", [("F16", 33), ("F16", 101), ("BF16", 64), ("U8", 37), ("U8", 3), ("F32", 1)])
def test_gather_dtypes_odd_rows(dev, dtype, dim):
    d = getattr(dgz, dtype)
    R = dim * dgz.ELEM_BYTES[d]
    rows = 2000
    t = HostTable(rows, R, seed=dim, base=dgz.ELEM_BYTES[d] * 3, dtype=d)
    try:
        idx = gen.random_ids(rows, 555, seed=dim)
        want, _ = oracle.gather(t.np, R, idx)
        for variant in (1, 4, 2, 3):
            for off in (0, dgz.ELEM_BYTES[d]):
                got = _gather_dev(t, idx, cfg=dgz.gather_cfg(variant=variant), out_offset=off)
                assert np.array_equal(got, want), (variant, off)
    finally:
        t.close()


def test_gather_edge_cases(dev):
    R, rows = 520, 1000
    t = HostTable(rows, R, seed=3)
    try:
        # n = 0 is a no-op
        assert _gather_dev(t, np.zeros(0, np.int64)).shape == (0, R)
        # n = 1, first and last row (span ends at the registered range), duplicates, int32 IDs
        for idx in (np.array([0]), np.array([rows - 1]), np.array([5, 5, 5, rows - 1, 0, 5])):
            want, _ = oracle.gather(t.np, R, idx)
            assert np.array_equal(_gather_dev(t, idx), want)
            assert np.array_equal(_gather_dev(t, idx, idx_dtype=torch.int32), want)
        # device-resident count: only the first m rows are written
        idx = gen.random_ids(rows, 300, 1)
        n_dev = torch.tensor([123], dtype=torch.int64, device="cuda")
        got = _gather_dev(t, idx, n_dev=n_dev, cfg=dgz.gather_cfg())
        want, _ = oracle.gather(t.np, R, idx[:123])
        assert np.array_equal(got[:123], want) and (got[123:] == 0xAB).all()
        # bounded persistent grids (the SM-partition knob) give the same bytes
        want, _ = oracle.gather(t.np, R, idx)
        for k in (1, 2, 8, 148):
            for variant in (1, 4):
                assert np.array_equal(_gather_dev(t, idx, cfg=dgz.gather_cfg(variant=variant, sm_count=k)), want)
    finally:
        t.close()


def test_gather_out_of_range_is_latched(dev):
    R, rows = 256, 100
    t = HostTable(rows, R, seed=4)
    try:
        idx = np.array([1, rows, 2, -1, rows - 1], dtype=np.int64)
        for variant in (1, 4, 2):
            got = _gather_dev(t, idx, cfg=dgz.gather_cfg(variant=variant))
            with pytest.raises(dgz.RangeError):
                dgz.check_errors(t.table)
            dgz.check_errors(t.table)  # the flag is cleared by the check
            want, _ = oracle.gather(t.np, R, idx)
            for r in (0, 2, 4):
                assert np.array_equal(got[r], want[r])
            assert (got[1] == 0xAB).all() and (got[3] == 0xAB).all()
    finally:
        t.close()


def test_gather_invalid_args(dev):
    t = HostTable(10, 64, seed=1, dtype=dgz.F32)
    try:
        idx = torch.zeros(4, dtype=torch.int64, device="cuda")
        out = torch.empty(4 * 64 + 4, dtype=torch.uint8, device="cuda")
        with pytest.raises(dgz.DgzError) as e:
            dgz.gather(t.table, idx, out[1:], n=4)  # not aligned to the fp32 element
        assert e.value.status == dgz.ERR_INVALID
        with pytest.raises(dgz.DgzError) as e:
            dgz.gather(t.table, idx, out, n=-1)
        assert e.value.status == dgz.ERR_INVALID
    finally:
        t.close()


def test_registration_info(dev):
    t = HostTable(1000, 512, seed=2, base=64)
    try:
        info = t.table.info
        assert info.rows == 1000 and info.row_bytes == 512 and info.base_mod128 == 64 and info.elem_bytes == 1
        assert info.pinned_bytes >= 1000 * 512
    finally:
        t.close()


# ------------------------------------------------------------------------------------------------
# sampler parity
# ------------------------------------------------------------------------------------------------
def _sample_dev(off, col, seeds, fanouts, rng_seed, col64=False):
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col.astype(np.int64 if col64 else np.int32)).cuda())
    bufs = dgz.SampleBuffers(g.n_nodes, max(len(seeds), 1), fanouts)
    s = torch.from_numpy(np.asarray(seeds, dtype=np.int64)).cuda()
    dgz.sample_uniform(g, s, fanouts, rng_seed, bufs)
    torch.cuda.synchronize()
    return g, bufs


def _compare_plan(off, col, seeds, fanouts, rng_seed, col64=False):
    want = oracle.sample_uniform(off, col, seeds, fanouts, rng_seed)
    g, bufs = _sample_dev(off, col, seeds, fanouts, rng_seed, col64)
    sizes = bufs.sizes_host.tolist()
    assert sizes == want.sizes.tolist()
    assert bufs.sizes_dev.cpu().tolist() == sizes
    assert np.array_equal(bufs.ids[:sizes[-1]].cpu().numpy(), want.U)
    n = sizes[-1]
    srt = bufs.ids_sorted[:n].cpu().numpy()
    assert np.array_equal(srt, np.sort(want.U))
    assert np.array_equal(want.U[bufs.ids_sorted_pos[:n].cpu().numpy()], srt)
    for k, (nbr, cnt, loc) in enumerate(bufs.hop_blocks()):
        assert np.array_equal(cnt.cpu().numpy(), want.cnt[k])
        assert np.array_equal(nbr.cpu().numpy(), want.nbr[k])
        assert np.array_equal(loc.cpu().numpy(), want.local[k])
    return want, bufs


@pytest.mark.parametrize("cid", [1])
def test_sampler_config1_many_batches(dev, cid):
    c = gen.CONFIGS[cid]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    for j in range(12):  # crosses an epoch boundary (10 batches per epoch), short last batch
        seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
        _compare_plan(off, col, seeds, c.fanouts, gen.batch_rng_seed(c.seed, j))


@pytest.mark.parametrize("n,deg,fan", [(20_000, 50.5, (15, 10, 5)), (5_000, 492.0, (25, 10)), (300_000, 14.4, (15, 10, 5)),
                                       (1000, 3.0, (64, 1, 0, 2)), (70_000, 8.0, ())])
def test_sampler_shapes(dev, n, deg, fan):
    off, col = gen.gen_csr(n, deg, n)
    seeds = gen.batch_seeds(n, 1024 if n > 1024 else n // 2, n, 3)
    _compare_plan(off, col, seeds, fan, gen.batch_rng_seed(n, 3))
    _compare_plan(off, col, seeds, fan, gen.batch_rng_seed(n, 3), col64=True)


def test_sampler_seed_cases(dev):
    off, col = gen.gen_csr(3000, 6.0, 5)
    _compare_plan(off, col, [7, 3, 7, 9, 3, 2999, 0], (4, 3), 99)      # duplicates: first kept
    _compare_plan(off, col, [1], (10,), 5)
    # n_seeds = 0
    g, bufs = _sample_dev(off, col, [], (3, 2), 1)
    assert bufs.sizes_host.tolist() == [0, 0, 0]
    # out-of-range seed: latched, reported by dgz_sample_check, the seed is dropped
    g, bufs = _sample_dev(off, col, [5, 3000, 6], (2,), 1)
    with pytest.raises(dgz.RangeError):
        dgz.sample_check(bufs)
    assert bufs.ids[:2].cpu().tolist() == [5, 6]


def test_sampler_isolated_and_large_seed_set(dev):
    off = np.zeros(50_001, dtype=np.int64)
    col = np.zeros(0, dtype=np.int32)
    _compare_plan(off, col, gen.batch_seeds(50_000, 9000, 1, 0), (5, 5), 3)
    off, col = gen.gen_csr(200_000, 4.0, 8)
    _compare_plan(off, col, gen.batch_seeds(200_000, 20_000, 8, 1), (3, 2), 4)   # > one seed chunk
    for ns in (4095, 4096, 4097, 6000):                                          # one-block / multi-kernel seed paths
        seeds = gen.batch_seeds(200_000, ns, 8, 2)
        seeds[5] = seeds[3]                                                       # a duplicate
        _compare_plan(off, col, seeds, (2,), 6)


def test_sample_then_gather_device_count(dev):
    """The step as the bench runs it: sampler -> gather with the device-resident |U|."""
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, 0)
        rs = gen.batch_rng_seed(c.seed, 0)
        g, bufs = _sample_dev(off, col, seeds, c.fanouts, rs)
        L = len(c.fanouts)
        out = torch.empty(bufs.bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
        dgz.gather(t.table, bufs.ids, out, n=bufs.bounds[-1], n_dev=bufs.sizes_dev[L:L + 1], cfg=dgz.gather_cfg())
        torch.cuda.synchronize()
        want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
        n = want.U.shape[0]
        exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
        assert np.array_equal(out[:n * c.row_bytes].cpu().numpy().reshape(n, -1), exp)
    finally:
        t.close()


@pytest.mark.parametrize("variant", [1, 4])
@pytest.mark.parametrize("sched", [0, 1, 2])
@pytest.mark.parametrize("R,base", [(512, 0), (400, 16), (2408, 8), (100, 4), (20, 0)])
def test_gather_perm(dev, variant, sched, R, base):
    rows = 4000
    t = HostTable(rows, R, seed=R + 99, base=base, dtype=dgz.F32)
    try:
        idx = gen.random_ids(rows, 1500 + 7, seed=R)
        want, _ = oracle.gather(t.np, R, idx)
        order = np.argsort(idx, kind="stable")
        ids_s = torch.from_numpy(idx[order]).cuda()
        pos_s = torch.from_numpy(order.astype(np.int64)).cuda()
        out = torch.full((idx.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        for sms in (0, 3, 64):
            out.fill_(0xAB)
            dgz.gather_perm(t.table, ids_s, pos_s, out, cfg=dgz.gather_cfg(variant=variant, schedule=sched, sm_count=sms))
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), sms
    finally:
        t.close()


@pytest.mark.parametrize("cid", [1, 3])
def test_step_sorted_gather_matches_oracle(dev, cid):
    """The bench step: GPU sampler (sorted outputs) -> dgz_gather_perm with the device count."""
    c = gen.CONFIGS[cid]
    n_nodes = c.n_nodes
    off, col = gen.gen_csr(n_nodes, c.avg_degree, c.seed)
    t = HostTable(n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        for j in (0, 5):
            seeds = gen.batch_seeds(n_nodes, c.batch, c.seed, j)
            rs = gen.batch_rng_seed(c.seed, j)
            g, bufs = _sample_dev(off, col, seeds, c.fanouts, rs)
            L = len(c.fanouts)
            out = torch.empty(bufs.bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
            dgz.gather_perm(t.table, bufs.ids_sorted, bufs.ids_sorted_pos, out, n=bufs.bounds[-1],
                            n_dev=bufs.sizes_dev[L:L + 1])
            torch.cuda.synchronize()
            want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
            n = want.U.shape[0]
            exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
            assert np.array_equal(out[:n * c.row_bytes].cpu().numpy().reshape(n, -1), exp)
    finally:
        t.close()


@pytest.mark.parametrize("R,sms,warps,n", [(4096, 4, 8, 6000), (16384, 2, 4, 1500), (65536, 1, 4, 300), (512, 1, 2, 50000),
                                            # more consumer warps than ring slots, or S not a multiple of
                                            # them (jobs j and j + S must share a consumer)
                                            (40960, 2, 0, 700), (65536, 2, 0, 500), (8192, 2, 32, 4000),
                                            (20000, 1, 8, 900), (30000, 3, 5, 800)])
def test_bulk_ring_wraparound(dev, R, sms, warps, n):
    """BULK: many more rows per CTA than ring slots (slot reuse across many mbarrier phases),
    rows up to 64 KiB (ring of 3 slots), rows ending exactly at the end of the registered table."""
    rows = max(n // 2, 8)
    t = HostTable(rows, R, seed=R + n, dtype=dgz.F32)
    try:
        idx = np.concatenate([np.arange(rows, dtype=np.int64), gen.random_ids(rows, n - rows, seed=R)])
        want, _ = oracle.gather(t.np, R, idx)
        for flags in (0,):
            got = _gather_dev(t, idx, cfg=dgz.gather_cfg(variant=dgz.GATHER_BULK, sm_count=sms, warps_per_cta=warps))
            assert np.array_equal(got, want)
    finally:
        t.close()


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 8, 16, 26, 32, 34])
def test_segment_flags(dev, flags):   # 1 = NO_MERGE (a no-op without dst_pos), 2 = DEEP, 8/16 = L2 cache hints
    R, rows = 520, 5000
    t = HostTable(rows, R, seed=flags, base=8, dtype=dgz.F32)
    try:
        idx = gen.random_ids(rows, 3000, seed=flags)
        want, _ = oracle.gather(t.np, R, idx)
        for sms, warps in ((0, 0), (3, 2), (148, 16)):
            got = _gather_dev(t, idx, cfg=dgz.gather_cfg(sm_count=sms, warps_per_cta=warps, flags=flags))
            assert np.array_equal(got, want)
    finally:
        t.close()


def test_fetch_on_green_context_partition(dev):
    """The same bytes when sampling + gather run on a green-context SM partition (step a6)."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        ng, per = dgz.partition_groups()
        assert ng * per <= 148 and per >= 1
        for flags, groups in ((dgz.PARTITION_SPREAD, None), (dgz.PARTITION_FINE, None), (0, None),
                              (0, [ng - 1, 3, 7, 20]), (0, list(range(10, 18)))):   # explicit SM groups
            part = dgz.Partition(8, -1, flags, groups=groups)
            assert part.fetch_sms >= 8 and part.fetch_sms + part.compute_sms <= 148
            if groups is not None:
                assert part.fetch_sms == len(groups) * per
            # flags == 0 case: the sampler on a second stream of the fetch SMs (dgz_partition_stream), so sampling
            # j+1 overlaps gathering j on the same partition
            sstream = part.stream(0, -1) if (flags == 0 and groups is None) else None
            f = MinibatchFetcher(t.table, g, c.fanouts, c.batch, fetch_stream=part.fetch_stream, sample_stream=sstream)
            for j in (0, 3):
                seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
                rs = gen.batch_rng_seed(c.seed, j)
                mb = f.fetch(torch.from_numpy(seeds).pin_memory(), rs)
                n = mb.sizes()[-1]
                want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
                exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
                assert np.array_equal(mb.bufs.ids[:n].cpu().numpy(), want.U)
                assert np.array_equal(mb.rows[:n].cpu().numpy(), exp)
            del f
            part.destroy()
    finally:
        t.close()


@pytest.mark.parametrize("R,n", [(512, 5000), (100, 777), (2408, 3000), (64, 1)])
def test_order_ids_then_gather_perm(dev, R, n):
    """Arbitrary ID lists (duplicates, out of range) -> dgz_order_ids -> dgz_gather_perm."""
    rows = 4000
    t = HostTable(rows, R, seed=R + 5, dtype=dgz.F32)
    try:
        idx = gen.random_ids(rows, n, seed=n)
        if n > 10:
            idx[3] = idx[7]          # duplicate
        ids = torch.from_numpy(idx).cuda()
        srt, pos = dgz.order_ids(ids, rows)
        torch.cuda.synchronize()
        assert np.array_equal(srt.cpu().numpy(), np.sort(idx))
        assert np.array_equal(idx[pos.cpu().numpy()], srt.cpu().numpy())
        out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
        dgz.gather_perm(t.table, srt, pos, out)
        torch.cuda.synchronize()
        want, _ = oracle.gather(t.np, R, idx)
        assert np.array_equal(out.cpu().numpy().reshape(n, R), want)
        if n > 10:   # an out-of-range ID is kept once and reported by the gather
            idx2 = idx.copy()
            idx2[5] = rows + 3
            srt, pos = dgz.order_ids(torch.from_numpy(idx2).cuda(), rows)
            assert sorted(srt.cpu().tolist()) == sorted(idx2.tolist())
            dgz.gather_perm(t.table, srt, pos, out)
            with pytest.raises(dgz.RangeError):
                dgz.check_errors(t.table)
    finally:
        t.close()


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("R,base", [(512, 0), (400, 16), (2408, 8), (100, 4)])
def test_hot_row_cache_gather(dev, G, R, base):
    """NEXT-1 HBM row cache: cached rows from HBM shards, the rest by zero-copy; same bytes."""
    rows = 5000
    t = HostTable(rows, R, seed=R + G, base=base, dtype=dgz.F32)
    try:
        hot = gen.distinct_ids(rows, 700, seed=G)
        cache = dgz.HotRowCache(t.table, torch.from_numpy(hot).cuda(), n_shards=G)
        torch.cuda.synchronize()
        dgz.check_errors(t.table)
        sm = cache.slot_map.cpu().numpy()
        assert (sm[hot] == np.arange(700)).all() and (np.delete(sm, hot) == -1).all()
        for g in range(G):   # shard g row k = table[hot[g + k*G]]
            k = np.arange(g, 700, G)
            want, _ = oracle.gather(t.np, R, hot[k])
            assert np.array_equal(cache.shards[g][:k.shape[0]].cpu().numpy(), want)
        idx = np.concatenate([gen.random_ids(rows, 2000, seed=R), hot[:300]])
        want, _ = oracle.gather(t.np, R, idx)
        out = torch.full((idx.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        cache.gather(torch.from_numpy(idx).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
        o = np.argsort(idx, kind="stable")
        out.fill_(0xAB)
        cache.gather(torch.from_numpy(idx[o]).cuda(), out, dst_pos=torch.from_numpy(o.astype(np.int64)).cuda(),
                     cfg=dgz.gather_cfg(sm_count=5, warps_per_cta=2))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    finally:
        t.close()


def test_device_table_and_empty_cache(dev):
    R, rows = 512, 3000
    t = HostTable(rows, R, seed=11, dtype=dgz.F32)
    try:
        dev_copy = torch.from_numpy(t.np.copy()).cuda()
        dt = dgz.DeviceTable(dev_copy.data_ptr(), rows, R // 4, dgz.F32)
        assert dt.info.flags & dgz.REG_DEVICE
        idx = gen.random_ids(rows, 1000, seed=2)
        want, _ = oracle.gather(t.np, R, idx)
        out = torch.empty(1000 * R, dtype=torch.uint8, device="cuda")
        dgz.gather(dt, torch.from_numpy(idx).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
        dt.unregister()
        cache = dgz.HotRowCache(t.table, torch.zeros(0, dtype=torch.int64, device="cuda"))
        out.zero_()
        cache.gather(torch.from_numpy(idx).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    finally:
        t.close()


def test_host_allocation_kinds(dev):
    """Every host-table allocation kind registers and gathers the same bytes; VMM export/import
    maps the same pages at a second address."""
    import os as _os
    R, rows = 512, 4096
    nbytes = R * rows
    idx = gen.random_ids(rows, 700, seed=5)
    kinds = [("anon", dgz.HOST_HUGEPAGE), ("cudapin", dgz.HOST_CUDA_PINNED), ("vmm", dgz.HOST_VMM)]
    for name, flags in kinds:
        buf = dgz.HostBuffer(nbytes, flags=flags)
        host = buf.numpy(0, nbytes)
        gen.fill_table(buf.ptr, nbytes, 17)
        t = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
        want, _ = oracle.gather(host, R, idx)
        out = torch.empty(700 * R, dtype=torch.uint8, device="cuda")
        dgz.gather(t.table if hasattr(t, "table") else t, torch.from_numpy(idx).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), name
        if name == "vmm":
            assert t.info.flags & dgz.REG_VMM_BACKED
            fd = buf.export_fd()
            b2 = dgz.HostBuffer(nbytes, import_fd=fd)
            assert b2.ptr != buf.ptr and np.array_equal(b2.numpy(0, 4096), host[:4096])
            b2.free()
            _os.close(fd)
        t.unregister()
        buf.free()


@pytest.mark.parametrize("variant", [1, 4])
def test_gather_flag_order(dev, variant):
    """DGZ_GATHER_FLAG_ORDER: sort on the device, gather in address order, scatter back."""
    R, rows = 400, 6000
    t = HostTable(rows, R, seed=21, base=16, dtype=dgz.F32)
    try:
        idx = gen.random_ids(rows, 5000, seed=4)
        idx[10] = idx[20]
        want, _ = oracle.gather(t.np, R, idx)
        got = _gather_dev(t, idx, cfg=dgz.gather_cfg(variant=variant, flags=dgz.FLAG_ORDER))
        assert np.array_equal(got, want)
        bad = idx.copy()
        bad[7] = rows + 1
        got = _gather_dev(t, bad, cfg=dgz.gather_cfg(variant=variant, flags=dgz.FLAG_ORDER))
        with pytest.raises(dgz.RangeError):
            dgz.check_errors(t.table)
        assert (got[7] == 0xAB).all() and np.array_equal(got[8:], want[8:])
    finally:
        t.close()


@pytest.mark.parametrize("graphs,sampler_sms", [(True, 0), (False, 0), (False, 8)])
def test_fetcher_modes_match_oracle(dev, graphs, sampler_sms):
    """MinibatchFetcher in CUDA-graph mode (device-resident sampler seed), sequential mode and the
    green-context sampler partition all give the oracle's minibatches, step after step."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        f = MinibatchFetcher(t.table, g, c.fanouts, c.batch, graphs=graphs, sampler_sms=sampler_sms)
        for j in (0, 1, 2, 3, 9):          # j = 9 is the short last batch of the epoch (eager path)
            seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
            rs = gen.batch_rng_seed(c.seed, j)
            mb = f.fetch(torch.from_numpy(seeds).cuda(), rs)
            n = mb.sizes()[-1]
            want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
            exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
            assert np.array_equal(mb.bufs.ids[:n].cpu().numpy(), want.U), j
            assert np.array_equal(mb.rows[:n].cpu().numpy(), exp), j
            f.release(mb)
        f.close()
    finally:
        t.close()


@pytest.mark.parametrize("R,base", [(400, 0), (520, 8), (512, 4), (512, 0), (2408, 0), (132, 64), (128, 16), (100, 4)])
@pytest.mark.parametrize("flags", [0, 1, 2, 24, 32, 34])
def test_gather_perm_adjacent_rows_merge(dev, R, base, flags):
    """Sorted lists full of table-adjacent rows: the shared 128 B line of two adjacent rows is
    fetched once and stored to both (MERGE), chains of adjacent rows, batch boundaries, and the
    NO_MERGE flag -- byte-identical to the oracle in every case."""
    rows = 6000
    t = HostTable(rows, R, seed=R + base, base=base, dtype=dgz.F32)
    try:
        runs = [np.arange(s, s + ln) for s, ln in ((0, 40), (100, 3), (777, 64), (2000, 1), (2002, 5), (5990, 10))]
        idx = np.unique(np.concatenate(runs + [gen.random_ids(rows, 900, seed=R)]))
        rng = np.random.default_rng(R)
        shuffled = idx[rng.permutation(idx.shape[0])]
        want, _ = oracle.gather(t.np, R, shuffled)
        order = np.argsort(shuffled, kind="stable")
        ids_s = torch.from_numpy(shuffled[order]).cuda()
        pos_s = torch.from_numpy(order.astype(np.int64)).cuda()
        out = torch.full((shuffled.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        for sms in (0, 3):
            out.fill_(0xAB)
            dgz.gather_perm(t.table, ids_s, pos_s, out, cfg=dgz.gather_cfg(sm_count=sms, flags=flags))
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy().reshape(-1, R), want), sms
        # cached rows in consecutive shard slots merge the same way
        hot = torch.from_numpy(np.arange(770, 900, dtype=np.int64)).cuda()
        cache = dgz.HotRowCache(t.table, hot)
        out.fill_(0xAB)
        cache.gather(ids_s, out, dst_pos=pos_s, cfg=dgz.gather_cfg(flags=flags))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    finally:
        t.close()


@pytest.mark.parametrize("R,rows,n,shape", [(128, 4_000_000, 3000, ("half", 1)),     # > 150 KiB apart
                                            (128, 400_000, 60_000, ("all", 1)),      # dense small rows
                                            (400, 2_000_000, 5000, ("half", 1)),     # 4 lines, > 150 KiB apart
                                            (400, 2_000_000, 8000, ("all", 1)),      # 4 lines, 100 KiB apart
                                            (400, 200_000, 80_000, ("all", 2)),      # 4 lines, dense
                                            (1028, 600_000, 2000, ("all", 2)),       # >= 8 lines
                                            (64, 8_000_000, 1000, ("half", 1))])
def test_gather_perm_default_launch_shapes(dev, R, rows, n, shape):
    """Every branch of the sorted gather's default launch-shape rule (row width x sparsity): the
    plan dgz_gather_plan reports, and the same bytes as the oracle."""
    t = HostTable(rows, R, seed=R + n, base=4, dtype=dgz.F32)
    try:
        plan = dgz.gather_plan(t.table, n, True)
        nsm = dgz.device_sm_count()
        assert (plan["sm_count"], plan["warps_per_cta"]) == ((nsm if shape[0] == "all" else nsm // 2), shape[1]), plan
        assert plan["line_loads_per_lane"] == 16 and plan["variant"] == "segment"
        idx = gen.random_ids(rows, n, seed=n)
        want, _ = oracle.gather(t.np, R, idx)
        srt, pos = dgz.order_ids(torch.from_numpy(idx).cuda(), rows)
        out = torch.full((n * R,), 0xAB, dtype=torch.uint8, device="cuda")
        dgz.gather_perm(t.table, srt, pos, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(n, R), want)
        dgz.check_errors(t.table)
    finally:
        t.close()


def test_tune_fetch_partition_then_fetch(dev):
    """pipeline.tune_fetch_partition times candidate partitions and returns the fastest; a fetch on
    it is byte-identical to the oracle."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher, tune_fetch_partition
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(2)]
        rs = [gen.batch_rng_seed(c.seed, j) for j in range(2)]
        ng, per = dgz.partition_groups()
        cands = [{"sms": 8, "flags": dgz.PARTITION_SPREAD}, {"groups": list(range(0, 8))}]
        part, cfg, res = tune_fetch_partition(t.table, g, c.fanouts, c.batch, seeds, rs, candidates=cands)
        assert len(res) == 2 and all(gbs > 0 for _, gbs in res)
        assert part.fetch_sms in (r[0]["fetch_sms"] for r in res)
        part.destroy()
        # under load: a stand-in consumer (a few HBM passes over the rows) on the compute SMs

        def consumer(mb, stream):
            with torch.cuda.stream(stream):
                for _ in range(4):
                    mb.rows.float().sum()
        part, cfg, res = tune_fetch_partition(t.table, g, c.fanouts, c.batch, seeds, rs,
                                              candidates=[dict(x, warps=2) for x in cands], consumer=consumer)
        assert len(res) == 2 and all(ms > 0 for _, ms in res) and cfg.warps_per_cta == 2
        f = MinibatchFetcher(t.table, g, c.fanouts, c.batch, fetch_stream=part.fetch_stream, gather_cfg=cfg)
        seeds_np = gen.batch_seeds(c.n_nodes, c.batch, c.seed, 5)
        mb = f.fetch(torch.from_numpy(seeds_np).cuda(), gen.batch_rng_seed(c.seed, 5))
        n = mb.sizes()[-1]
        want = oracle.sample_uniform(off, col, seeds_np, c.fanouts, gen.batch_rng_seed(c.seed, 5), with_blocks=False)
        exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
        assert np.array_equal(mb.bufs.ids[:n].cpu().numpy(), want.U)
        assert np.array_equal(mb.rows[:n].cpu().numpy(), exp)
        del f
        part.destroy()
    finally:
        t.close()


@pytest.mark.parametrize("R,base", [(8 << 20, 0), ((8 << 20) + 36, 4), ((32 << 20) - 4, 8)])
def test_gather_very_large_rows(dev, R, base):
    """Rows up to the SEGMENT limit (< 32 MiB per row): every line of every row, unsorted and
    sorted, at aligned and misaligned bases; 32 MiB rows are refused synchronously."""
    rows = 6
    t = HostTable(rows, R, seed=R % 1000, base=base, dtype=dgz.F32)
    try:
        idx = np.array([3, 0, 5, 3], dtype=np.int64)
        want, _ = oracle.gather(t.np, R, idx)
        assert np.array_equal(_gather_dev(t, idx), want)
        order = np.argsort(idx, kind="stable")
        out = torch.full((idx.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        dgz.gather_perm(t.table, torch.from_numpy(idx[order]).cuda(), torch.from_numpy(order.astype(np.int64)).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    finally:
        t.close()


def test_gather_refuses_rows_of_32_mib(dev):
    R = 32 << 20
    buf = dgz.HostBuffer(R + 4096)
    t = dgz.register_table(buf.ptr, 1, R // 4, dgz.F32)
    try:
        out = torch.empty(R, dtype=torch.uint8, device="cuda")
        with pytest.raises(dgz.DgzError):
            dgz.gather(t, torch.zeros(1, dtype=torch.int64, device="cuda"), out)
    finally:
        t.unregister()
        buf.free()


def test_sampler_limits(dev):
    """DGZ_MAX_LAYERS hops, DGZ_MAX_FANOUT on high-degree nodes (Floyd with f = 64), and every node
    of the graph as a seed (U = all nodes)."""
    off, col = gen.gen_csr(30_000, 100.0, 77)
    _compare_plan(off, col, gen.batch_seeds(30_000, 64, 77, 0), (dgz.MAX_FANOUT,), 5)
    _compare_plan(off, col, gen.batch_seeds(30_000, 16, 77, 1), (2,) * dgz.MAX_LAYERS, 6)
    off, col = gen.gen_csr(5000, 6.0, 78)
    _compare_plan(off, col, np.arange(5000, dtype=np.int64)[::-1].copy(), (3, 2), 7)


def test_concurrent_streams(dev):
    """Two samplers and two gathers (one with the work-counter schedule) in flight at once on two
    streams over the same graph and table: both minibatches equal the oracle's."""
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        bufs = [dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts) for _ in range(2)]
        outs = [torch.empty(bufs[0].bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
        L = len(c.fanouts)
        js = (2, 7)
        for k in range(2):
            s = streams[k]
            seeds = torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, js[k])).to("cuda", non_blocking=True)
            s.wait_stream(torch.cuda.current_stream())
            dgz.sample_uniform(g, seeds, c.fanouts, gen.batch_rng_seed(c.seed, js[k]), bufs[k], stream=s)
            b = bufs[k]
            dgz.gather_perm(t.table, b.ids_sorted, b.ids_sorted_pos, outs[k], n=b.bounds[-1], n_dev=b.sizes_dev[L:L + 1],
                            cfg=dgz.gather_cfg(flags=dgz.FLAG_DYNAMIC if k else 0), stream=s)
        torch.cuda.synchronize()
        for k in range(2):
            seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, js[k])
            want = oracle.sample_uniform(off, col, seeds, c.fanouts, gen.batch_rng_seed(c.seed, js[k]), with_blocks=False)
            n = want.U.shape[0]
            exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
            assert np.array_equal(bufs[k].ids[:n].cpu().numpy(), want.U)
            assert np.array_equal(outs[k][:n * c.row_bytes].cpu().numpy().reshape(n, -1), exp)
        dgz.check_errors(t.table)
    finally:
        t.close()


def test_calibrated_fetcher(dev):
    """pipeline.calibrated_fetcher times the pipelined and the sequential fetcher and keeps the faster;
    its minibatches equal the oracle's."""
    from paper_2103_03330_b200.pipeline import calibrated_fetcher
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = HostTable(c.n_nodes, c.row_bytes, seed=c.seed, dtype=dgz.F32)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        seeds = [torch.from_numpy(gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)).cuda() for j in range(3)]
        rs = [gen.batch_rng_seed(c.seed, j) for j in range(3)]
        f, choice = calibrated_fetcher(t.table, g, c.fanouts, c.batch, seeds, rs)
        assert choice["chosen"] == f.mode
        for j in (4, 5):
            seeds_np = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
            mb = f.fetch(torch.from_numpy(seeds_np).cuda(), gen.batch_rng_seed(c.seed, j))
            n = mb.sizes()[-1]
            want = oracle.sample_uniform(off, col, seeds_np, c.fanouts, gen.batch_rng_seed(c.seed, j), with_blocks=False)
            exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
            assert np.array_equal(mb.bufs.ids[:n].cpu().numpy(), want.U)
            assert np.array_equal(mb.rows[:n].cpu().numpy(), exp)
        f.close()
    finally:
        t.close()


def test_gather_plan_reports_table_kind_defaults(dev):
    """dgz_gather_plan: HBM-resident tables get 8 warps x 8 CTAs per SM; a host table's unsorted
    gather 16 warps; explicit configs are passed through."""
    nsm = dgz.device_sm_count()
    dev_rows = torch.empty(1000 * 512, dtype=torch.uint8, device="cuda")
    dt = dgz.DeviceTable(dev_rows.data_ptr(), 1000, 128, dgz.F32)
    try:
        p = dgz.gather_plan(dt, 1_000_000, False)
        assert (p["sm_count"], p["warps_per_cta"]) == (nsm, 8) and p["ctas"] == nsm * 8
        p = dgz.gather_plan(dt, 100_000, False)       # small lists: no more CTAs than 8-warp batches
        assert p["ctas"] == -(-(-(-100_000 // 32)) // 8)
    finally:
        dt.unregister()
    t = HostTable(1000, 512, seed=1, dtype=dgz.F32)
    try:
        p = dgz.gather_plan(t.table, 100_000, False)
        assert (p["sm_count"], p["warps_per_cta"], p["line_loads_per_lane"]) == (nsm, 16, 8)
        p = dgz.gather_plan(t.table, 100_000, True, dgz.gather_cfg(sm_count=12, warps_per_cta=4, flags=dgz.FLAG_DYNAMIC))
        assert (p["sm_count"], p["warps_per_cta"], p["schedule"]) == (12, 4, "work counter")
    finally:
        t.close()
