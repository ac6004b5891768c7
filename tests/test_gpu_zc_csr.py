"""Zero-copy CSR: the sampler reads a CSR left in pinned, mapped host memory
(dgz.HostGraph) by PCIe loads.  Same bar as the HBM CSR: sampled IDs, per-hop sizes, blocks and the
sorted order bit-exact against the oracle; gathered rows byte for byte."""
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


def _compare(off, col, seeds, fanouts, rs, offsets_in_hbm=True, managed=False):
    want = oracle.sample_uniform(off, col, seeds, fanouts, rs)
    g = dgz.HostGraph(off, col, offsets_in_hbm=offsets_in_hbm, managed=managed)
    try:
        bufs = dgz.SampleBuffers(g.n_nodes, max(len(seeds), 1), fanouts)
        dgz.sample_uniform(g, torch.from_numpy(np.asarray(seeds, dtype=np.int64)).cuda(), fanouts, rs, bufs)
        torch.cuda.synchronize()
        sizes = bufs.sizes_host.tolist()
        assert sizes == want.sizes.tolist()
        n = sizes[-1]
        assert np.array_equal(bufs.ids[:n].cpu().numpy(), want.U)
        assert np.array_equal(bufs.ids_sorted[:n].cpu().numpy(), np.sort(want.U))
        for k, (nbr, cnt, loc) in enumerate(bufs.hop_blocks()):
            assert np.array_equal(cnt.cpu().numpy(), want.cnt[k])
            assert np.array_equal(nbr.cpu().numpy(), want.nbr[k])
            assert np.array_equal(loc.cpu().numpy(), want.local[k])
    finally:
        g.close()


@pytest.mark.parametrize("n,deg,fan,col64", [(10_000, 10.0, (10, 5), False), (20_000, 50.5, (15, 10, 5), True),
                                             (5_000, 492.0, (25, 10), False), (1000, 3.0, (64, 1, 0, 2), False),
                                             (300_000, 14.4, (15, 10, 5), False)])
def test_zero_copy_csr_sampler(dev, n, deg, fan, col64):
    off, col = gen.gen_csr(n, deg, n + 1)
    if col64:
        col = col.astype(np.int64)
    for j, in_hbm, managed in ((0, True, False), (5, False, False), (7, True, True), (9, False, True)):
        # offsets in HBM (default) or also on the host; registered or managed host memory
        seeds = gen.batch_seeds(n, min(1024, n // 2), n + 1, j)
        _compare(off, col, seeds, fan, gen.batch_rng_seed(n + 1, j), offsets_in_hbm=in_hbm, managed=managed)


def test_zero_copy_csr_edge_cases(dev):
    off = np.zeros(4001, dtype=np.int64)                     # no edges at all: cols may be NULL
    for in_hbm in (True, False):
        _compare(off, np.zeros(0, dtype=np.int32), [5, 17, 3999, 5], (3, 2), 9, in_hbm)
    off, col = gen.gen_csr(3000, 6.0, 5)
    _compare(off, col, [7, 3, 7, 9, 3, 2999, 0], (4, 3), 99, False)


def test_zero_copy_csr_fetch_config3(dev):
    """The bench's fetch path (MinibatchFetcher: sampler on an 8-SM partition, sorted gather) with
    both the CSR and the feature table in host memory, products-shaped at full size."""
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    c = gen.CONFIGS[3]
    R = c.row_bytes
    buf = dgz.HostBuffer(c.table_bytes + 4096)
    gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    g = dgz.HostGraph(off, col)
    try:
        f = MinibatchFetcher(table, g, c.fanouts, c.batch)
        host = buf.numpy(0, c.table_bytes)
        for j in (1, 2):
            seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
            rs = gen.batch_rng_seed(c.seed, j)
            mb = f.fetch(torch.from_numpy(seeds).cuda(), rs)
            sizes = mb.sizes()
            want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
            assert sizes == want.sizes.tolist()
            n = sizes[-1]
            assert np.array_equal(mb.bufs.ids[:n].cpu().numpy(), want.U)
            exp = np.empty(n * R, dtype=np.uint8)
            assert oracle.gather_into(host.ctypes.data, c.n_nodes, R, want.U, exp) == 0
            assert np.array_equal(mb.rows[:n].cpu().numpy().reshape(-1), exp)
        f.close()
        dgz.check_errors(table)
    finally:
        g.close()
        table.unregister()
        buf.free()
