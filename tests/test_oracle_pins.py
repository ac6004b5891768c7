"""Pins of the CPU oracle against things other than itself (no GPU).

Each test checks the oracle against the paper's worked examples, SPEC special cases, a
published known-answer table, exact enumeration, or an independent brute-force recomputation
written here with Python sets/Counters.  See DESIGN.md "Oracle pins".
"""
from collections import Counter
from itertools import combinations

import numpy as np
import pytest

import dgz_inputs as gen
import oracle
from oracle import request_model as rm
from conftest import golden_lines


# --------------------------------------------------------------------------------------------
# Philox4x32-10: Random123 known-answer vectors (tests/golden/philox4x32_10_kat.txt)
# --------------------------------------------------------------------------------------------
def test_philox_kat():
    n = 0
    for line in golden_lines("philox4x32_10_kat.txt"):
        w = [int(x, 16) for x in line.split()]
        assert oracle.philox4x32_10(w[0:4], w[4:6]) == tuple(w[6:10])
        n += 1
    assert n == 3


# --------------------------------------------------------------------------------------------
# Uniform selection without replacement (Floyd): exact enumeration of subsets
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,f", [(5, 2), (6, 3), (7, 1), (8, 7), (4, 3)])
def test_select_uniform_subsets(d, f):
    """Every f-subset of d slots is equally likely (chi-square over many counter keys)."""
    M = 24000
    counts = Counter()
    for u in range(M):
        pos = oracle.select_positions(d, f, 0x1234567, 0, u)
        assert len(pos) == f and pos == sorted(pos) and len(set(pos)) == f
        assert all(0 <= p < d for p in pos)
        counts[tuple(pos)] += 1
    subsets = list(combinations(range(d), f))
    assert set(counts) == set(subsets)
    exp = M / len(subsets)
    chi2 = sum((counts[s] - exp) ** 2 / exp for s in subsets)
    dof = len(subsets) - 1
    # mean dof, sd sqrt(2 dof): 6 sigma bound (deterministic inputs, so no flakiness)
    assert chi2 < dof + 6 * (2 * dof) ** 0.5 + 10, chi2


def test_select_small_degree_takes_all():
    for d in range(0, 12):
        assert oracle.select_positions(d, 12, 99, 1, 5) == list(range(d))
    assert oracle.select_positions(5, 0, 1, 0, 0) == []


def test_select_counter_keyed():
    """Selection is a function of (seed, hop, node): different keys decorrelate."""
    a = [tuple(oracle.select_positions(1000, 10, 7, 0, u)) for u in range(50)]
    b = [tuple(oracle.select_positions(1000, 10, 7, 1, u)) for u in range(50)]
    c = [tuple(oracle.select_positions(1000, 10, 8, 0, u)) for u in range(50)]
    assert a == [tuple(oracle.select_positions(1000, 10, 7, 0, u)) for u in range(50)]
    assert sum(x == y for x, y in zip(a, b)) == 0 and sum(x == y for x, y in zip(a, c)) == 0


# --------------------------------------------------------------------------------------------
# Layered sampling: brute-force invariants on tiny graphs (north_star)
# --------------------------------------------------------------------------------------------
def _adj(off, col, u):
    return col[off[u]:off[u + 1]].tolist()


def _check_plan(off, col, seeds, fanouts, res):
    U = res.U.tolist()
    sizes = res.sizes.tolist()
    # unique, seeds (first occurrence) are the prefix
    assert len(U) == len(set(U))
    dedup = list(dict.fromkeys(np.asarray(seeds).tolist()))
    assert U[:len(dedup)] == dedup and sizes[0] == len(dedup)
    for k, f in enumerate(fanouts):
        nk = sizes[k]
        hop_ids = []
        for i in range(nk):
            u = U[i]
            adj = _adj(off, col, u)
            c = int(res.cnt[k][i])
            assert c == min(f, len(adj))                      # cardinality
            got = res.nbr[k][i][:c].tolist()
            assert all(x == -1 for x in res.nbr[k][i][c:].tolist())
            # sampled slots are distinct CSR slots: multiset inclusion
            assert not (Counter(got) - Counter(adj))          # membership
            if len(adj) <= f:
                assert got == adj                             # all slots, CSR order
            hop_ids += got
            assert [U[j] for j in res.local[k][i][:c].tolist()] == got
        new = sorted(set(hop_ids) - set(U[:nk]))              # frontier union
        assert U[nk:sizes[k + 1]] == new
    assert sizes[-1] == len(U)


@pytest.mark.parametrize("n,deg,fan,seed", [(50, 3.0, (4, 2), 1), (200, 8.0, (5, 3, 2), 2),
                                             (30, 20.0, (25,), 3), (1000, 2.0, (10, 10, 10), 4)])
def test_sampler_bruteforce(n, deg, fan, seed):
    off, col = gen.gen_csr(n, deg, seed)
    seeds = gen.batch_seeds(n, min(16, n), seed, 0)
    res = oracle.sample_uniform(off, col, seeds, fan, gen.batch_rng_seed(seed, 0))
    _check_plan(off, col, seeds, fan, res)
    # determinism
    res2 = oracle.sample_uniform(off, col, seeds, fan, gen.batch_rng_seed(seed, 0))
    assert np.array_equal(res.U, res2.U)
    # int64 column indices give the same plan
    res3 = oracle.sample_uniform(off, col.astype(np.int64), seeds, fan, gen.batch_rng_seed(seed, 0))
    assert np.array_equal(res.U, res3.U)


def test_sampler_order_independent_per_node():
    """A node's hop-0 sample depends only on (seed, hop, node), not its position."""
    off, col = gen.gen_csr(500, 30.0, 9)
    seeds = gen.batch_seeds(500, 40, 9, 0)
    a = oracle.sample_uniform(off, col, seeds, (5,), 77)
    b = oracle.sample_uniform(off, col, seeds[::-1].copy(), (5,), 77)
    ma = {int(u): a.nbr[0][i].tolist() for i, u in enumerate(a.U[:a.sizes[0]])}
    mb = {int(u): b.nbr[0][i].tolist() for i, u in enumerate(b.U[:b.sizes[0]])}
    assert ma == mb
    assert sorted(a.U.tolist()) == sorted(b.U.tolist())


def test_sampler_duplicate_seeds_keep_first():
    off, col = gen.gen_csr(100, 5.0, 3)
    res = oracle.sample_uniform(off, col, [7, 3, 7, 9, 3], (3,), 5)
    assert res.U[:3].tolist() == [7, 3, 9]
    _check_plan(off, col, [7, 3, 7, 9, 3], (3,), res)


def test_sampler_spec_cases():
    lines = dict(l.split(None, 1) for l in golden_lines("spec_sampler_cases.txt"))
    # star graph
    edges = [tuple(map(int, e.split(":"))) for e in lines["star_edges"].split(",")]
    n = 4
    off = np.zeros(n + 1, dtype=np.int64)
    for s, _ in edges:
        off[s + 1] += 1
    off = np.cumsum(off)
    col = np.array([d for _, d in sorted(edges)], dtype=np.int32)
    res = oracle.sample_uniform(off, col, [0], (10,), 42)
    expect = [int(x) for x in lines["star_expected"].split(",")]
    assert sorted(res.nbr[0][0][:res.cnt[0][0]].tolist()) == expect
    assert res.U.tolist() == [0] + expect
    # empty fanouts
    res = oracle.sample_uniform(off, col, [2, 1, 2], (), 1)
    assert res.U.tolist() == [2, 1] and res.sizes.tolist() == [2]
    # cycle
    n = 100
    off = np.arange(n + 1, dtype=np.int64) * 2
    col = np.array([[(u + 1) % n, (u - 1) % n] for u in range(n)], dtype=np.int32).reshape(-1)
    r1 = oracle.sample_uniform(off, col, [0], (1, 1), 42)
    r2 = oracle.sample_uniform(off, col, [0], (1, 1), 42)
    assert np.array_equal(r1.U, r2.U)
    _check_plan(off, col, [0], (1, 1), r1)


def test_sampler_seed_out_of_range():
    off, col = gen.gen_csr(10, 2.0, 1)
    with pytest.raises(IndexError):
        oracle.sample_uniform(off, col, [3, 10], (2,), 1)


def test_sampler_isolated_nodes():
    off = np.zeros(6, dtype=np.int64)
    col = np.zeros(0, dtype=np.int32)
    res = oracle.sample_uniform(off, col, [4, 0], (3, 3), 1)
    assert res.U.tolist() == [4, 0] and res.cnt[0].tolist() == [0, 0]


# --------------------------------------------------------------------------------------------
# Gather: closed form out[r] = table[idx[r]]
# --------------------------------------------------------------------------------------------
@pytest.mark.parametrize("rows,R", [(100, 512), (37, 400), (50, 2408), (64, 3), (10, 1), (9, 4096)])
def test_gather_equals_take(rows, R):
    table = gen.table_bytes(rows * R, 11)
    idx = gen.random_ids(rows, 300, 5)
    out, bad = oracle.gather(table, R, idx)
    assert bad == 0
    assert np.array_equal(out, np.take(table.reshape(rows, R), idx, axis=0))
    # brute force: every gathered row equals table[id], byte for byte
    for r in (0, 17, 299):
        assert bytes(out[r]) == bytes(table[idx[r] * R:(idx[r] + 1) * R])


def test_gather_out_of_range_and_empty():
    table = gen.table_bytes(10 * 8, 1)
    out, bad = oracle.gather(table, 8, [1, 10, -1, 9])
    assert bad == 2
    assert bytes(out[0]) == bytes(table[8:16]) and bytes(out[3]) == bytes(table[72:80])
    assert not out[1].any() and not out[2].any()
    out, bad = oracle.gather(table, 8, [])
    assert out.shape == (0, 8) and bad == 0


# --------------------------------------------------------------------------------------------
# Request model: the paper's worked examples (tests/golden/paper_requests.txt)
# --------------------------------------------------------------------------------------------
def test_paper_request_examples():
    n = 0
    for line in golden_lines("paper_requests.txt"):
        name, feat, idx, base, shift, expect = line.split()
        cnt, _ = rm.listing2_requests([int(idx)], int(feat), 4, base=int(base), shift=bool(int(shift)))
        assert cnt == int(expect), name
        n += 1
    assert n == 4


def test_fig5_histograms_and_segment_plan():
    # unshifted / shifted histograms of the P:437-447 example (SURVEY 4 item 3 erratum of S:228)
    assert rm.listing2_requests([1], 120, shift=False)[1] == {96: 3, 64: 1, 32: 4}
    assert rm.listing2_requests([1], 120, shift=True)[1] == {128: 3, 64: 1, 32: 1}
    # the segment plan reaches the same 5 requests on this example
    assert rm.segment_plan_requests([1], 480)[0] == 5


def test_segment_plan_is_row_minimum():
    """Per-row closed forms agree with byte enumeration; the plan never loses to Listing 2."""
    for R in (16, 48, 100, 128, 132, 400, 480, 516, 1028, 2408):
        for o in range(0, 128, 4):
            addrs = range(o, o + R)
            assert rm.row_lines(o, R) == len({a // 128 for a in addrs})
            assert rm.row_sectors(o, R) == len({a // 32 for a in addrs})
    rng = np.random.default_rng(0)
    for feat in (33, 100, 120, 150, 257):
        for _ in range(5):
            ids = rng.choice(10000, size=6, replace=False).tolist()
            plan = rm.segment_plan_requests(ids, feat * 4)[0]
            assert plan == sum(rm.row_lines(i * feat * 4, feat * 4) for i in ids)
            assert plan <= rm.listing2_requests(ids, feat, shift=True)[0]
            assert plan <= rm.listing2_requests(ids, feat, shift=False)[0]


def test_merged_plan_never_exceeds_listing2():
    """With the shared line of table-adjacent rows fetched once, the segment plan issues no more
    requests than Listing 2 even on dense sorted lists (where Listing 2's flat enumeration merges
    such lines too), and exactly the per-row minimum when no two rows are adjacent."""
    rng = np.random.default_rng(1)
    for feat in (33, 100, 120, 130, 602):
        R = feat * 4
        for _ in range(6):
            ids = sorted(set(rng.integers(0, 60, size=20).tolist()))      # dense: many adjacent IDs
            merged = rm.merged_plan_requests(ids, R)
            assert merged <= rm.segment_plan_requests(ids, R)[0]
            assert merged <= rm.listing2_requests(ids, feat, shift=True)[0]
            assert merged <= rm.listing2_requests(ids, feat, shift=False)[0]
        sparse = [i * 7 for i in range(20)]                                  # no adjacent rows
        assert rm.merged_plan_requests(sparse, R) == rm.segment_plan_requests(sparse, R)[0]


def test_merged_plan_sectors_brute_force():
    """merged_plan_sectors = distinct 32 B sectors per batch, checked by enumerating every byte
    address of every row; equals the per-row sector sum when no two rows of a batch share a sector."""
    rng = np.random.default_rng(2)
    for R in (100, 128, 400, 516, 2408):
        for base in (0, 4, 64):
            ids = sorted(set(rng.integers(0, 90, size=40).tolist()))
            want = 0
            for b0 in range(0, len(ids), 32):
                want += len({(base + i * R + k) // 32 for i in ids[b0:b0 + 32] for k in range(R)})
            assert rm.merged_plan_sectors(ids, R, base) == want
            sparse = [i * 9 for i in range(50)]
            assert rm.merged_plan_sectors(sparse, R, base) == sum(rm.row_sectors(base + i * R, R) for i in sparse)


# ----------------------------------------------------------------------------------------------
# The consumer's layer: oracle.sage_mean_linear
# ----------------------------------------------------------------------------------------------
def _mat(s, conv=float):
    return np.array([[conv(v) for v in row.split(",")] for row in s.split(";")])


def test_sage_layer_worked_example():
    """The hand-worked example in tests/golden/sage_layer_example.txt."""
    from fractions import Fraction
    g = dict(l.split(None, 1) for l in golden_lines("sage_layer_example.txt"))
    x, w = _mat(g["x"]), _mat(g["w"])
    local, cnt = _mat(g["local"], int), np.array([int(v) for v in g["cnt"].split(",")])
    want = _mat(g["y"], lambda v: float(Fraction(v)))
    got = oracle.sage_mean_linear(x, local, cnt, w)
    assert np.allclose(got, want, rtol=0, atol=1e-15)


def test_sage_layer_is_dense_normalised_adjacency_product():
    """Y equals the paper's matrix form A_hat . H . W^T with A_hat built explicitly as a dense
    [n_dst, n_src] matrix (self edge + one entry per sampled slot, repeated IDs adding up, rows
    scaled by 1/(1+cnt)), on random blocks; and the two degenerate cases: no samples and W = I
    give Y = H[:n_dst]; every row sampling itself f times with W = I gives Y = H[:n_dst]."""
    rng = np.random.default_rng(11)
    for n_src, n_dst, dim, hidden, f in ((40, 12, 5, 3, 4), (200, 64, 17, 32, 7), (9, 9, 1, 1, 3)):
        x = rng.standard_normal((n_src, dim))
        w = rng.standard_normal((hidden, dim))
        cnt = rng.integers(0, f + 1, size=n_dst)
        local = np.full((n_dst, f), -1, dtype=np.int64)
        A = np.zeros((n_dst, n_src))
        for i in range(n_dst):
            local[i, :cnt[i]] = rng.integers(0, n_src, size=cnt[i])
            A[i, i] += 1.0
            for q in range(cnt[i]):
                A[i, local[i, q]] += 1.0
            A[i] /= 1.0 + cnt[i]
        assert np.allclose(oracle.sage_mean_linear(x, local, cnt, w), A @ x @ w.T, rtol=1e-12, atol=1e-12)
        eye = np.eye(dim)
        assert np.array_equal(oracle.sage_mean_linear(x, local, np.zeros(n_dst, np.int64), eye), x[:n_dst])
        selfs = np.repeat(np.arange(n_dst)[:, None], f, axis=1)
        assert np.allclose(oracle.sage_mean_linear(x, selfs, np.full(n_dst, f), eye), x[:n_dst], rtol=1e-14, atol=1e-14)
