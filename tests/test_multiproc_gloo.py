"""N > 1 host-side logic on CPU with gloo, world_size 2 (no GPU): the shared host table (one
copy created by rank 0 in /dev/shm, mapped by every rank: P:616-627), the seed partition
j = i*G + rank, rank-independent minibatches, and the max-over-ranks timing rule."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, memfd=False):
    try:
        os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                           "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                           "DGZ_BENCH_FORCE_MEMFD": "1" if memfd else "0"})
        sys.path.insert(0, ROOT)
        import bench
        import dgz_inputs as gen
        import oracle
        from paper_2103_03330_b200 import dgz

        d = bench.Dist(world)
        cfg = gen.CONFIGS[1]
        buf, _ = bench.make_table(cfg, d, dgz)
        host = buf.numpy()[:cfg.table_bytes]
        ok_table = bool(np.array_equal(host[::977], gen.table_bytes(cfg.table_bytes, cfg.seed)[::977]))
        K = 3
        mine = [i * world + rank for i in range(K)]
        off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed)
        off2, col2, e2, csr_bufs = bench.make_csr(cfg, d, dgz)          # one CSR per box in /dev/shm
        ok_csr = bool(e2 == off[-1] and np.array_equal(off2, off) and np.array_equal(col2, col))
        sizes = []
        for j in mine:
            s = oracle.sample_uniform(off, col, gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j), cfg.fanouts,
                                      gen.batch_rng_seed(cfg.seed, j), with_blocks=False)
            sizes.append(int(s.U.shape[0]))
        tot, = d.allreduce([float(sum(sizes))], "sum")
        mx, = d.allreduce([float(rank + 1)], "max")
        d.barrier()
        buf.free()
        for b in csr_bufs:
            b.free()
        d.close()
        q.put((rank, ok_table and ok_csr, mine, sizes, tot, mx))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("memfd", [False, True])   # shared objects in /dev/shm, or rank 0's memfds (short /dev/shm)
def test_two_ranks_share_table_and_partition_batches(memfd):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q, memfd)) for r in range(2)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=240)
        assert len(r) == 6, r
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    assert res[0][1] and res[1][1]                                   # both ranks see the same table and CSR bytes
    assert sorted(res[0][2] + res[1][2]) == list(range(6))           # j = i*G + rank: disjoint cover
    assert res[0][4] == res[1][4] == sum(res[0][3]) + sum(res[1][3])  # all-reduce SUM of bytes
    assert res[0][5] == res[1][5] == 2.0                              # MAX over ranks
    # a batch's sample does not depend on which rank draws it (keyed by global batch j)
    import dgz_inputs as gen
    import oracle
    cfg = gen.CONFIGS[1]
    off, col = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed)
    j = res[1][2][0]
    s = oracle.sample_uniform(off, col, gen.batch_seeds(cfg.n_nodes, cfg.batch, cfg.seed, j), cfg.fanouts,
                              gen.batch_rng_seed(cfg.seed, j), with_blocks=False)
    assert s.U.shape[0] == res[1][3][0]
