"""Round-2 parity gaps (VERDICT r1 "Next round" 1), CUDA path vs oracle-derived expectations.

1. The stand-in consumer ``dgz_aggregate_mean`` (P:554-555 fig:singlegpu):
   y[i] = (x[i] + sum_q x[local[i, q]]) * (1 / (1 + cnt[i])), q < cnt[i], fp32, summed in the
   order q = 0, 1, ...  The expected value is computed here in numpy from the ORACLE's gathered
   rows (``oracle.gather`` of the oracle's U) and the ORACLE's per-hop ``local`` / ``cnt`` blocks
   (``oracle.sample_uniform``), one fp32 rounding per add as the kernel does, so the comparison
   is bit-exact (IEEE fp32 add / multiply / correctly rounded division; the library is built
   without fast-math).
2. The address-sorted MERGE path (``dgz_order_ids`` + ``dgz_gather_perm``, what bench and the
   config-5 sweeps time) over every config-5 row width x base offset, on lists dense in
   table-adjacent rows (so sorted neighbours share 128 B lines and the merge is exercised),
   against ``oracle.gather`` byte for byte.
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


class FloatTable:
    """A registered host table of finite fp32 values (rows x dim) at byte offset ``base``."""

    def __init__(self, rows, dim, seed, base=0):
        self.rows, self.dim, self.R = rows, dim, dim * 4
        self.buf = dgz.HostBuffer(rows * self.R + base + 4096)
        raw = self.buf.numpy()
        vals = gen.float_table(rows * dim, seed)
        raw[base:base + rows * self.R] = vals.view(np.uint8)
        self.np = raw[base:base + rows * self.R]
        self.table = dgz.register_table(self.buf.ptr + base, rows, dim, dgz.F32)

    def close(self):
        self.table.unregister()
        self.buf.free()


def expected_mean(x, local, cnt):
    """Sequential fp32 mean over {self} + sampled neighbours, the kernel's order (see module doc)."""
    nk = cnt.shape[0]
    acc = x[:nk].copy()
    f = local.shape[1] if local.ndim == 2 else 0
    for q in range(f):
        m = cnt > q
        acc[m] = acc[m] + x[local[m, q]]
    inv = (np.float32(1.0) / (np.float32(1.0) + cnt.astype(np.float32))).astype(np.float32)
    return (acc * inv[:, None]).astype(np.float32)


def _gpu_minibatch(t, off, col, seeds, fanouts, rs):
    g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
    bufs = dgz.SampleBuffers(g.n_nodes, len(seeds), fanouts)
    dgz.sample_uniform(g, torch.from_numpy(seeds).cuda(), fanouts, rs, bufs)
    L = len(fanouts)
    rows = torch.empty((bufs.bounds[-1], t.dim), dtype=torch.float32, device="cuda")
    dgz.gather_perm(t.table, bufs.ids_sorted, bufs.ids_sorted_pos, rows, n=bufs.bounds[-1],
                    n_dev=bufs.sizes_dev[L:L + 1])
    torch.cuda.synchronize()
    return g, bufs, rows


@pytest.mark.parametrize("n_nodes,deg,dim,fanouts,batch", [
    (10_000, 10.0, 128, (10, 5), 1024),        # config 1
    (60_000, 50.5, 100, (15, 10, 5), 512),     # products-shaped degree, 400 B rows
    (5_000, 40.0, 37, (7, 3), 300),            # dim not a multiple of 32
])
def test_aggregate_mean_matches_oracle(dev, n_nodes, deg, dim, fanouts, batch):
    off, col = gen.gen_csr(n_nodes, deg, n_nodes + dim)
    t = FloatTable(n_nodes, dim, seed=dim * 7 + 1)
    try:
        for j in (0, 3):
            seeds = gen.batch_seeds(n_nodes, batch, n_nodes, j)
            rs = gen.batch_rng_seed(n_nodes, j)
            want = oracle.sample_uniform(off, col, seeds, fanouts, rs)
            xw, bad = oracle.gather(t.np, t.R, want.U)
            assert bad == 0
            xw = xw.view(np.float32).reshape(-1, dim)
            g, bufs, rows = _gpu_minibatch(t, off, col, seeds, fanouts, rs)
            n = int(want.sizes[-1])
            assert np.array_equal(rows[:n].cpu().numpy(), xw)            # the consumer's input
            for k, (nbr, cnt, loc) in enumerate(bufs.hop_blocks()):
                nk = int(want.sizes[k])
                exp = expected_mean(xw, want.local[k], want.cnt[k])
                for repeat, sms, cps in ((1, 0, 0), (3, 0, 0), (2, 8, 2), (1, 148, 1)):
                    y = torch.full((bufs.bounds[k] + 3, dim), float("nan"), dtype=torch.float32, device="cuda")
                    dgz.aggregate_mean(rows.view(-1), dim, loc.reshape(-1), cnt, fanouts[k], bufs.sizes_dev[k:k + 1],
                                       bufs.bounds[k], y, repeat=repeat, sm_count=sms, ctas_per_sm=cps)
                    torch.cuda.synchronize()
                    got = y.cpu().numpy()
                    assert np.array_equal(got[:nk].view(np.uint32), exp.view(np.uint32)), (k, repeat, sms, cps)
                    assert np.isnan(got[nk:]).all()                        # rows past |F_k| untouched
    finally:
        t.close()


def test_aggregate_mean_on_oracle_inputs(dev):
    """The kernel alone, fed the oracle's rows and blocks (no GPU sampler or gather upstream);
    n_dst from the host bound (no device count), and an empty destination set."""
    n_nodes, dim, fanouts = 3_000, 64, (6, 4)
    off, col = gen.gen_csr(n_nodes, 12.0, 77)
    t = FloatTable(n_nodes, dim, seed=5)
    try:
        seeds = gen.batch_seeds(n_nodes, 200, 77, 1)
        want = oracle.sample_uniform(off, col, seeds, fanouts, 1234)
        xw, _ = oracle.gather(t.np, t.R, want.U)
        xw = xw.view(np.float32).reshape(-1, dim)
        x = torch.from_numpy(xw.copy()).cuda()
        for k, f in enumerate(fanouts):
            nk = int(want.sizes[k])
            loc = torch.from_numpy(np.ascontiguousarray(want.local[k].astype(np.int32))).cuda()
            cnt = torch.from_numpy(np.ascontiguousarray(want.cnt[k].astype(np.int32))).cuda()
            y = torch.empty((nk, dim), dtype=torch.float32, device="cuda")
            dgz.aggregate_mean(x.view(-1), dim, loc.view(-1), cnt, f, None, nk, y)
            torch.cuda.synchronize()
            exp = expected_mean(xw, want.local[k], want.cnt[k])
            assert np.array_equal(y.cpu().numpy().view(np.uint32), exp.view(np.uint32))
        y = torch.zeros((1, dim), dtype=torch.float32, device="cuda")
        dgz.aggregate_mean(x.view(-1), dim, loc.view(-1), cnt, 4, None, 0, y)   # n_dst = 0: no-op
        torch.cuda.synchronize()
        assert (y == 0).all()
    finally:
        t.close()


class ByteTable:
    def __init__(self, rows, R, seed, base, dtype):
        eb = dgz.ELEM_BYTES[dtype]
        self.R = R
        self.buf = dgz.HostBuffer(rows * R + base + 4096)
        arr = self.buf.numpy()
        gen.fill_table(arr.ctypes.data + base, rows * R, seed)
        self.np = arr[base:base + rows * R]
        self.table = dgz.register_table(self.buf.ptr + base, rows, R // eb, dtype)

    def close(self):
        self.table.unregister()
        self.buf.free()


@pytest.mark.parametrize("R", gen.SWEEP_ROW_BYTES)
@pytest.mark.parametrize("base", gen.SWEEP_BASE_OFFSETS)
def test_sorted_merge_path_sweep(dev, R, base):
    """dgz_order_ids + dgz_gather_perm (line merge on) at every config-5 width x base offset, on
    dense runs of table-adjacent rows with duplicates and a ragged tail; the bench's whole-GPU
    default launch and the overlap sweep's small-partition launch (work counter, 16 loads)."""
    rows = max(64, min(4000, (8 << 20) // R))
    for dtype in (dgz.U8, dgz.F32):
        t = ByteTable(rows, R, seed=R * 7 + base, base=base, dtype=dtype)
        try:
            idx = gen.adjacent_run_ids(rows, 1000 + 17, seed=R + base)
            want, bad = oracle.gather(t.np, R, idx)
            assert bad == 0
            ids = torch.from_numpy(idx).cuda()
            srt, pos = dgz.order_ids(ids, rows)
            for cfg in (None, dgz.gather_cfg(sm_count=8, warps_per_cta=4, flags=dgz.FLAG_DEEP | dgz.FLAG_DYNAMIC)):
                out = torch.full((idx.shape[0] * R + 16,), 0xAB, dtype=torch.uint8, device="cuda")
                dgz.gather_perm(t.table, srt, pos, out, cfg=cfg)
                torch.cuda.synchronize()
                got = out.cpu().numpy()
                assert np.array_equal(got[:idx.shape[0] * R].reshape(-1, R), want), (dtype, cfg)
                assert (got[idx.shape[0] * R:] == 0xAB).all()
        finally:
            t.close()
