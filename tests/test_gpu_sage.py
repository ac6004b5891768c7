"""The stand-in consumer's layer ``dgz_sage_mean_linear`` (mean over each dst node's
sampled neighbours of the gathered rows, then a small GEMM -- on the tcgen05 tensor cores) against
the oracle's fp64 layer ``oracle.sage_mean_linear`` (P:225-227 Y = A_hat H W^T).

Two checks per output element (y[i, n], K = dim):
* against the oracle (the paper's layer in fp64): |y - Y| <= (2^-8 + 2^-14) * (mean|x| . |W|^T)[i, n].
  2^-8 is bf16's unit roundoff (h is rounded to bf16 before the product, |bf16(h) - h| <= 2^-8 |h|
  and |h_k| <= mean_k|x|); 2^-14 covers the fp32 mean (<= (cnt + 2) 2^-24 relative) and the fp32
  accumulation of K exact bf16 x bf16 products (K = 256 at most: <= 2^-16 relative to sum |h w|).
* against the kernel's own precision steps replayed in numpy from the ORACLE's inputs: h in fp32 in
  the kernel's order (bit-exact, as dgz_aggregate_mean's test shows), rounded to bf16 (round to nearest
  even), times W in fp64: |y - ref| <= 2^-16 * (|bf16(h)| . |W|^T) -- only the tensor core's fp32
  accumulation order is free.
A transposed operand, a wrong row, a dropped neighbour or a mis-laid core matrix moves y by O(|y|),
far outside both bounds.
"""
import numpy as np
import pytest
import torch

import dgz_inputs as gen
import oracle
from test_gpu_consumer_merge import FloatTable, _gpu_minibatch, expected_mean

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2103_03330_b200 import dgz


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)


def bf16_rne(a: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 (round to nearest even) -> fp32, for finite values."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def check_layer(y, x, local, cnt, w_bf16):
    """y: kernel output [n_dst, hidden] (numpy fp32); x [n_src, dim] fp32; local [n_dst, f]; cnt [n_dst];
    w_bf16: the torch bf16 weight [hidden, dim]."""
    n_dst = cnt.shape[0]
    w = w_bf16.float().cpu().numpy().astype(np.float64)
    aw = np.abs(w)
    want = oracle.sage_mean_linear(x, local, cnt, w)
    habs = oracle.sage_mean_linear(np.abs(x), local, cnt, np.eye(x.shape[1]))
    tol = (2.0 ** -8 + 2.0 ** -14) * (habs @ aw.T)
    err = np.abs(y.astype(np.float64) - want)
    assert (err <= tol).all(), f"vs oracle: worst excess {np.max(err - tol)} at {np.unravel_index(np.argmax(err - tol), err.shape)}"
    hb = bf16_rne(expected_mean(x.astype(np.float32), local, cnt)).astype(np.float64)
    ref = hb @ w.T
    tol2 = 2.0 ** -16 * (np.abs(hb) @ aw.T) + 1e-30
    err2 = np.abs(y.astype(np.float64) - ref)
    assert (err2 <= tol2).all(), f"vs bf16 replay: worst excess {np.max(err2 - tol2)}"
    assert y.shape[0] == n_dst


def _weight(hidden, dim, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(hidden, dim, generator=g) / np.sqrt(dim)).to(torch.bfloat16).cuda()


@pytest.mark.parametrize("n_nodes,deg,dim,hidden,fanouts,batch", [
    (10_000, 10.0, 128, 256, (10, 5), 1024),       # config 1 rows, hidden 256 (UMMA N max)
    (10_000, 10.0, 128, 64, (10, 5), 1024),
    (60_000, 50.5, 100, 128, (15, 10, 5), 512),    # products-shaped 400 B rows: K padded 100 -> 112
    (5_000, 40.0, 37, 48, (7, 3), 300),            # dim 37 (scalar loads, K 48), hidden 48
])
def test_sage_layer_on_sampled_minibatch(dev, n_nodes, deg, dim, hidden, fanouts, batch):
    """The GPU minibatch (sampler + zero-copy gather) feeds the layer, every hop; the expected values
    come from the oracle's sample and the oracle's gathered rows."""
    off, col = gen.gen_csr(n_nodes, deg, n_nodes + dim)
    t = FloatTable(n_nodes, dim, seed=dim * 7 + 3)
    w = _weight(hidden, dim, dim + hidden)
    try:
        seeds = gen.batch_seeds(n_nodes, batch, n_nodes, 1)
        rs = gen.batch_rng_seed(n_nodes, 1)
        want = oracle.sample_uniform(off, col, seeds, fanouts, rs)
        xw, bad = oracle.gather(t.np, t.R, want.U)
        assert bad == 0
        xw = xw.view(np.float32).reshape(-1, dim)
        g, bufs, rows = _gpu_minibatch(t, off, col, seeds, fanouts, rs)
        n = int(want.sizes[-1])
        assert np.array_equal(rows[:n].cpu().numpy(), xw)
        for k, (nbr, cnt, loc) in enumerate(bufs.hop_blocks()):
            nk = int(want.sizes[k])
            for repeat, sms, cps in ((1, 0, 0), (2, 0, 0), (3, 8, 1), (1, 148, 2)):
                y = torch.full((bufs.bounds[k] + 5, hidden), float("nan"), dtype=torch.float32, device="cuda")
                dgz.sage_mean_linear(rows.view(-1), dim, loc.reshape(-1), cnt, fanouts[k], bufs.sizes_dev[k:k + 1],
                                     bufs.bounds[k], w, y, repeat=repeat, sm_count=sms, ctas_per_sm=cps)
                torch.cuda.synchronize()
                got = y.cpu().numpy()
                check_layer(got[:nk], xw, want.local[k], want.cnt[k], w)
                assert np.isnan(got[nk:]).all(), (k, repeat, sms, cps)     # rows past |F_k| untouched
    finally:
        t.close()


@pytest.mark.parametrize("dim,hidden,fanout,n_dst", [
    (128, 256, 5, 172_000 // 16),   # config-4 last hop shape (|F_2| / 16), ragged tail
    (128, 16, 1, 1),                # one row, N = 16 (UMMA minimum)
    (256, 256, 40, 129),            # K = 256, fanout > 32 (indices past the warp shuffle)
    (200, 80, 3, 128),              # exactly one tile
    (64, 128, 10, 127),             # one short tile
    (16, 32, 2, 1000),
    (1, 16, 4, 300),                # dim 1: K padded 1 -> 16
    (602, 256, 25, 300),            # config-2 rows (602 fp32): K in 5 chunks of 128 accumulated in TMEM
    (320, 256, 5, 200),             # 3 chunks, the last one half padding
    (300, 64, 10, 257),             # hidden 64: chunks of 256 (the second mostly padding)
    (130, 48, 6, 400),              # dim 130: scalar loads (dim % 4 != 0), K 144 in one chunk
])
def test_sage_layer_shapes(dev, dim, hidden, fanout, n_dst):
    """Synthetic blocks (random positions, counts 0..fanout, repeated IDs allowed) over every tile
    shape: K padding, N from 16 to 256, ragged last tiles, fanout past 32."""
    rng = np.random.default_rng(dim * 1000 + hidden + fanout)
    n_src = n_dst + 3 * n_dst + 7
    x = rng.uniform(-1, 1, size=(n_src, dim)).astype(np.float32)
    cnt = rng.integers(0, fanout + 1, size=n_dst).astype(np.int32)
    local = np.full((n_dst, fanout), -1, dtype=np.int32)
    for i in range(n_dst):
        local[i, :cnt[i]] = rng.integers(0, n_src, size=cnt[i])
    w = _weight(hidden, dim, fanout)
    xd, ld, cd = torch.from_numpy(x).cuda(), torch.from_numpy(local).cuda(), torch.from_numpy(cnt).cuda()
    y = torch.full((n_dst, hidden), float("nan"), dtype=torch.float32, device="cuda")
    dgz.sage_mean_linear(xd.view(-1), dim, ld.view(-1), cd, fanout, None, n_dst, w, y)
    torch.cuda.synchronize()
    check_layer(y.cpu().numpy(), x, local, cnt, w)


def test_sage_layer_edges(dev):
    """n_dst = 0 is a no-op; a device count below the host bound leaves the rows past it untouched;
    hidden outside {16, 32, ..., 256} is refused (DGZ_ERR_INVALID); rows too wide for one shared-memory
    operand are chunked along K."""
    dim, hidden, f = 64, 32, 4
    x = torch.rand(500, dim, device="cuda")
    loc = torch.zeros(400, f, dtype=torch.int32, device="cuda")
    cnt = torch.ones(400, dtype=torch.int32, device="cuda")
    w = _weight(hidden, dim, 1)
    y = torch.zeros(400, hidden, device="cuda")
    dgz.sage_mean_linear(x.view(-1), dim, loc.view(-1), cnt, f, None, 0, w, y)
    torch.cuda.synchronize()
    assert (y == 0).all()
    n_dev = torch.tensor([200], dtype=torch.int64, device="cuda")
    y.fill_(float("nan"))
    dgz.sage_mean_linear(x.view(-1), dim, loc.view(-1), cnt, f, n_dev, 400, w, y)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    check_layer(got[:200], x.cpu().numpy(), loc[:200].cpu().numpy(), cnt[:200].cpu().numpy(), w)
    assert np.isnan(got[200:]).all()
    for bad_hidden in (8, 24, 272):
        with pytest.raises(dgz.DgzError):
            dgz.sage_mean_linear(x.view(-1), dim, loc.view(-1), cnt, f, None, 400, _weight(bad_hidden, dim, 2),
                                 torch.zeros(400, bad_hidden, device="cuda"))
    # wide rows are chunked along K (2 x 128 + a padded 64 here), not refused
    big = torch.rand(10, 320, device="cuda")
    yb = torch.zeros(10, 256, device="cuda")
    wb = _weight(256, 320, 3)
    dgz.sage_mean_linear(big.view(-1), 320, loc.view(-1), cnt, f, None, 10, wb, yb)
    torch.cuda.synchronize()
    check_layer(yb.cpu().numpy(), big.cpu().numpy(), loc[:10].cpu().numpy(), cnt[:10].cpu().numpy(), wb)
    assert dgz.sage_workspace(128, 256) == ((256 + 128) * 128 * 2 + 48, 256)
    assert dgz.sage_workspace(602, 256) == ((256 + 128) * 128 * 2 + 48, 256)     # K chunk 128
    assert dgz.sage_workspace(200, 64) == ((64 + 128) * 208 * 2 + 48, 64)        # one chunk


def test_sage_layer_full_size_config4(dev):
    """BASELINE config 4 at full size, in the launch configuration bench.py times: the fetcher's GPU minibatch
    (sampler + address-sorted zero-copy gather from the 56.9 GB table, here filled with finite fp32 values)
    feeds the layer on the last hop's block (|F_2| ~ 1.5e5 destination rows, fanout 5, 128 -> 256,
    non-persistent grid); 3000 random destination rows plus the first and last 64 are computed one by one
    by the oracle from ITS sample and ITS gather of the rows they need."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    c = gen.CONFIGS[4]
    dim, R, hidden = c.dim, c.row_bytes, 256
    buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table_f32(buf.ptr, c.n_nodes * dim, c.seed)
    table = dgz.register_table(buf.ptr, c.n_nodes, dim, dgz.F32)
    try:
        off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
        graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        f = MinibatchFetcher(table, graph, c.fanouts, c.batch)
        j = 3
        seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
        rs = gen.batch_rng_seed(c.seed, j)
        mb = f.fetch(torch.from_numpy(seeds).cuda(), rs)
        sizes = mb.sizes()
        L = len(c.fanouts)
        k = L - 1
        _, cnt_d, loc_d = mb.bufs.hop_blocks(sizes)[k]
        nk = sizes[k]
        w = _weight(hidden, dim, 44)
        y = torch.full((mb.bufs.bounds[k], hidden), float("nan"), dtype=torch.float32, device="cuda")
        dgz.sage_mean_linear(mb.rows.view(torch.float32).view(-1), dim, loc_d.reshape(-1), cnt_d, c.fanouts[k],
                             mb.bufs.sizes_dev[k:k + 1], mb.bufs.bounds[k], w, y)
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        assert np.isnan(got[nk:]).all()
        want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs)
        assert int(want.sizes[k]) == nk
        rng = np.random.default_rng(5)
        pick = np.unique(np.concatenate([rng.choice(nk, 3000, replace=False), np.arange(64), np.arange(nk - 64, nk)]))
        loc, cnt = want.local[k][pick], want.cnt[k][pick]
        # the rows these destinations read: themselves first (x_sub[i] = dst pick[i]), then their neighbours
        nbr_pos = np.unique(np.concatenate([loc[i, :cnt[i]] for i in range(len(pick))]))
        extra = np.setdiff1d(nbr_pos, pick)
        pos = np.concatenate([pick, extra])
        remap = {int(p): i for i, p in enumerate(pos)}
        loc_sub = np.full_like(loc, -1)
        for i in range(len(pick)):
            loc_sub[i, :cnt[i]] = [remap[int(p)] for p in loc[i, :cnt[i]]]
        host = buf.numpy(0, c.table_bytes)
        xs = np.empty(len(pos) * R, dtype=np.uint8)
        assert oracle.gather_into(host.ctypes.data, c.n_nodes, R, want.U[pos], xs) == 0
        check_layer(got[pick], xs.view(np.float32).reshape(-1, dim), loc_sub, cnt, w)
        dgz.check_errors(table)
    finally:
        table.unregister()
        buf.free()
