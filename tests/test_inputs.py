"""Input generators (dgz_inputs): determinism, bijective seed permutation, degree law."""
import numpy as np

import dgz_inputs as gen


def test_csr_deterministic_and_valid():
    off, col = gen.gen_csr(5000, 10.0, 3)
    off2, col2 = gen.gen_csr(5000, 10.0, 3)
    assert np.array_equal(off, off2) and np.array_equal(col, col2)
    assert off[0] == 0 and np.all(np.diff(off) >= 0) and off[-1] == col.shape[0]
    assert col.min() >= 0 and col.max() < 5000
    deg = np.diff(off)
    assert abs(deg.mean() - 10.0) < 0.3 and abs(deg.var() - 10.0) < 1.5   # Poisson: mean = var


def test_epoch_permutation_partitions_nodes():
    n, b = 10_007, 1000
    seen = np.concatenate([gen.batch_seeds(n, b, 5, j) for j in range(11)])
    assert seen.shape[0] == n and np.array_equal(np.sort(seen), np.arange(n))
    assert gen.batch_seeds(n, b, 5, 10).shape[0] == 7            # short last batch
    assert not np.array_equal(gen.batch_seeds(n, b, 5, 11), gen.batch_seeds(n, b, 5, 0))


def test_table_fill_keyed_by_position():
    a = gen.table_bytes(1000, 9)
    b = gen.table_bytes(2000, 9)
    assert np.array_equal(a, b[:1000]) and not np.array_equal(a, gen.table_bytes(1000, 10))


def test_rank_partition():
    world = 4
    owned = [gen.rank_batches(r, world, 5) for r in range(world)]
    flat = sorted(j for o in owned for j in o)
    assert flat == list(range(20)) and all(j % world == r for r, o in enumerate(owned) for j in o)


def test_fill_table_f32():
    """Finite keyed fp32 values on the 2^-23 grid of [-1, 1), deterministic in (seed, index), independent
    of the count filled (keyed by position) -- the recipe of the layer's full-size parity table."""
    a = np.empty(100_000, np.float32)
    gen.fill_table_f32(a, a.size, 7)
    assert np.isfinite(a).all() and a.min() >= -1.0 and a.max() < 1.0
    assert np.array_equal(a * np.float32(2 ** 23), np.round(a * np.float32(2 ** 23)))
    b = np.empty(1000, np.float32)
    gen.fill_table_f32(b, b.size, 7)
    assert np.array_equal(a[:1000], b)
    gen.fill_table_f32(b, b.size, 8)
    assert not np.array_equal(a[:1000], b)
    assert abs(float(a.mean())) < 0.01 and abs(float(a.std()) - 3 ** -0.5) < 0.01
