"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(MinibatchFetcher defaults: GPU sampler -> address-sorted dgz_gather_perm, device-resident |U|).
Every sampled ID list is compared exactly with the oracle's, and every gathered row byte for byte
with the oracle's gather of the same table."""
import numpy as np
import pytest
import torch

import dgz_inputs as gen
import oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_full_size_config(cid):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_03330_b200 import dgz
    from paper_2103_03330_b200.pipeline import MinibatchFetcher
    torch.cuda.set_device(0)
    c = gen.CONFIGS[cid]
    R = c.row_bytes
    buf = dgz.HostBuffer(c.table_bytes + 4096, flags=dgz.HOST_HUGEPAGE)
    gen.fill_table(buf.ptr, c.table_bytes, c.seed)
    table = dgz.register_table(buf.ptr, c.n_nodes, c.dim, dgz.F32)
    try:
        off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
        graph = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        f = MinibatchFetcher(table, graph, c.fanouts, c.batch)
        host = buf.numpy(0, c.table_bytes)
        for j in (0, 7):
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
        if c.table_bytes >= 4 << 30:
            # plain dgz_gather of a large unsorted list: fetched in address order internally
            idx = gen.random_ids(c.n_nodes, 100_000, seed=3)
            out = torch.empty(100_000 * R, dtype=torch.uint8, device="cuda")
            dgz.gather(table, torch.from_numpy(idx).cuda(), out)
            exp = np.empty(100_000 * R, dtype=np.uint8)
            oracle.gather_into(host.ctypes.data, c.n_nodes, R, idx, exp)
            assert np.array_equal(out.cpu().numpy(), exp)
        dgz.check_errors(table)
    finally:
        table.unregister()
        buf.free()


def test_output_beyond_4gib():
    """64-bit destination offsets: 10.5 M rows of 512 B (5.4 GB of output) gathered from a 2 GB
    table, unsorted and address-sorted; sampled rows (every 997th plus the last 64) byte-exact."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_03330_b200 import dgz
    torch.cuda.set_device(0)
    R, rows, n = 512, 4_000_000, 10_500_000
    buf = dgz.HostBuffer(rows * R + 4096)
    gen.fill_table(buf.ptr, rows * R, 99)
    table = dgz.register_table(buf.ptr, rows, R // 4, dgz.F32)
    try:
        idx_np = gen.random_ids(rows, n, seed=4)
        idx = torch.from_numpy(idx_np).cuda()
        out = torch.empty(n * R, dtype=torch.uint8, device="cuda")
        pick = np.concatenate([np.arange(0, n, 997), np.arange(n - 64, n)])
        exp = np.empty(pick.shape[0] * R, dtype=np.uint8)
        assert oracle.gather_into(buf.ptr, rows, R, idx_np[pick], exp) == 0
        exp = exp.reshape(-1, R)
        pk = torch.from_numpy(pick).cuda()
        dgz.gather(table, idx, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.view(n, R)[pk].cpu().numpy(), exp)
        srt, pos = dgz.order_ids(idx, rows)
        out.zero_()
        dgz.gather_perm(table, srt, pos, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.view(n, R)[pk].cpu().numpy(), exp)
        dgz.check_errors(table)
    finally:
        table.unregister()
        buf.free()
