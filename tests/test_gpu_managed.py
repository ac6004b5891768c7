"""The managed host table (DGZ_HOST_MANAGED: CUDA managed memory kept in host memory, mapped for the
GPU at registration) through the same kernels, byte for byte against the oracle: plain and
address-sorted gathers at several widths and base offsets, and the bench step (GPU sampler ->
dgz_gather_perm with the device count) on config 1."""
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


class ManagedTable:
    def __init__(self, rows, R, seed, base=0, dtype=None):
        dtype = dgz.F32 if dtype is None else dtype
        eb = dgz.ELEM_BYTES[dtype]
        self.buf = dgz.HostBuffer(rows * R + base + 4096, flags=dgz.HOST_MANAGED)
        gen.fill_table(self.buf.ptr + base, rows * R, seed)
        self.np = self.buf.numpy(base, rows * R)
        self.R = R
        self.table = dgz.register_table(self.buf.ptr + base, rows, R // eb, dtype)

    def close(self):
        self.table.unregister()
        self.buf.free()


@pytest.mark.parametrize("R,base", [(512, 0), (128, 0), (400, 16), (2408, 8), (100, 4), (1030, 2), (64, 64)])
def test_managed_gathers(dev, R, base):
    rows = 5000
    t = ManagedTable(rows, R, seed=R + base, base=base, dtype=dgz.F16 if R % 4 else dgz.F32)
    try:
        info = t.table.info
        assert info.flags & dgz.REG_MANAGED and info.dev_ptr == t.buf.ptr + base
        idx = gen.random_ids(rows, 1777, seed=R)
        want, _ = oracle.gather(t.np, R, idx)
        out = torch.full((idx.shape[0] * R,), 0xAB, dtype=torch.uint8, device="cuda")
        dgz.gather(t.table, torch.from_numpy(idx).cuda(), out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
        srt, pos = dgz.order_ids(torch.from_numpy(idx).cuda(), rows)
        out.fill_(0xAB)
        dgz.gather_perm(t.table, srt, pos, out)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().reshape(-1, R), want)
    finally:
        t.close()


def test_managed_step_matches_oracle(dev):
    c = gen.CONFIGS[1]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    t = ManagedTable(c.n_nodes, c.row_bytes, seed=c.seed)
    try:
        g = dgz.Graph(torch.from_numpy(off).cuda(), torch.from_numpy(col).cuda())
        bufs = dgz.SampleBuffers(c.n_nodes, c.batch, c.fanouts)
        L = len(c.fanouts)
        for j in (0, 4):
            seeds = gen.batch_seeds(c.n_nodes, c.batch, c.seed, j)
            rs = gen.batch_rng_seed(c.seed, j)
            dgz.sample_uniform(g, torch.from_numpy(seeds).cuda(), c.fanouts, rs, bufs)
            out = torch.empty(bufs.bounds[-1] * c.row_bytes, dtype=torch.uint8, device="cuda")
            dgz.gather_perm(t.table, bufs.ids_sorted, bufs.ids_sorted_pos, out, n=bufs.bounds[-1],
                            n_dev=bufs.sizes_dev[L:L + 1])
            torch.cuda.synchronize()
            want = oracle.sample_uniform(off, col, seeds, c.fanouts, rs, with_blocks=False)
            n = want.U.shape[0]
            exp, _ = oracle.gather(t.np, c.row_bytes, want.U)
            assert np.array_equal(out[:n * c.row_bytes].cpu().numpy().reshape(n, -1), exp)
        # the host copy is untouched by the GPU's reads (the pages stay where the CPU put them)
        assert np.array_equal(t.np[:4096], gen.table_bytes(4096, c.seed))
    finally:
        t.close()


def test_managed_alloc_refuses_a_name(dev):
    with pytest.raises(dgz.DgzError):
        dgz.HostBuffer(1 << 20, shm_name="/dgz_managed_named", flags=dgz.HOST_MANAGED)
