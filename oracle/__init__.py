"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, single-threaded CPU reference for the hot path of arXiv 2103.03330
(PyTorch-Direct): layered uniform neighbour sampling and the sparse
feature row gather (Listing 2).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this package.  It shares
no code with ``paper_2103_03330_b200`` (the CUDA path) and neither imports the other.

Pins (what checks this oracle against something other than itself) live in
``tests/test_oracle_pins.py``; every function below is pinned -- see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import request_model  # noqa: F401  (PCIe request-count model)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dgz_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", tmp, _SRC])
        os.replace(tmp, _SO)
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        vp, i64, i32, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
        L.oracle_philox4x32_10.argtypes = [vp, vp, vp]
        L.oracle_select_positions.argtypes = [i64, i32, u64, ctypes.c_int, i64, vp]
        L.oracle_select_positions.restype = i64
        L.oracle_sample_uniform.argtypes = [i64, vp, vp, ctypes.c_int, vp, i64, vp, ctypes.c_int, u64,
                                            vp, i64, vp, vp, i64, vp, i64, vp]
        L.oracle_sample_uniform.restype = ctypes.c_int
        L.oracle_gather.argtypes = [vp, i64, i64, vp, i64, vp]
        L.oracle_gather.restype = i64
        _lib = L
    return _lib


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"], "oracle needs contiguous arrays"
    return a.ctypes.data


def philox4x32_10(ctr, key) -> tuple:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    _L().oracle_philox4x32_10(_p(c), _p(k), _p(o))
    return tuple(int(x) for x in o)


def select_positions(d: int, f: int, rng_seed: int, hop: int, u: int) -> list:
    pos = np.zeros(max(f, 1) if d > f else max(d, 1), dtype=np.int64)
    c = _L().oracle_select_positions(d, f, rng_seed & (2**64 - 1), hop, u, _p(pos))
    return pos[:c].tolist()


class SampleResult:
    """U (frontier-prefix unique IDs), sizes |F_0..F_L|, per-hop nbr/cnt/local blocks."""

    def __init__(self, U, sizes, nbr, cnt, local):
        self.U, self.sizes, self.nbr, self.cnt, self.local = U, sizes, nbr, cnt, local


class OracleError(RuntimeError):
    pass


def sample_uniform(off: np.ndarray, col: np.ndarray, seeds, fanouts, rng_seed: int,
                   with_blocks: bool = True) -> SampleResult:
    off = np.ascontiguousarray(off, dtype=np.int64)
    col = np.ascontiguousarray(col)
    assert col.dtype in (np.int32, np.int64)
    n_nodes = off.shape[0] - 1
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.int64))
    fan = np.ascontiguousarray(np.asarray(fanouts, dtype=np.int32))
    L = int(fan.shape[0])
    ns = int(seeds.shape[0])
    # capacity: min(N, n_seeds * prod(1 + f))
    cap, b = min(n_nodes, ns), ns
    nbr_cap = cnt_cap = 0
    for f in fan.tolist():
        cnt_cap += min(n_nodes, b)
        nbr_cap += min(n_nodes, b) * f
        b *= 1 + f
        cap = min(n_nodes, b)
    cap = max(cap, 1)
    U = np.zeros(cap, dtype=np.int64)
    sizes = np.zeros(L + 1, dtype=np.int64)
    nbr = np.zeros(max(nbr_cap, 1), dtype=np.int64) if with_blocks else None
    cnt = np.zeros(max(cnt_cap, 1), dtype=np.int32) if with_blocks else None
    loc = np.zeros(max(nbr_cap, 1), dtype=np.int32) if with_blocks else None
    st = _L().oracle_sample_uniform(
        n_nodes, _p(off), _p(col), int(col.dtype == np.int64), _p(seeds) if ns else None, ns,
        _p(fan) if L else None, L, rng_seed & (2**64 - 1), _p(U), cap, _p(sizes),
        _p(nbr) if with_blocks else None, nbr_cap, _p(cnt) if with_blocks else None, cnt_cap,
        _p(loc) if with_blocks else None)
    if st == 4:
        raise IndexError("seed out of range")
    if st != 0:
        raise OracleError(f"oracle_sample_uniform status {st}")
    n = int(sizes[-1]) if L >= 0 else 0
    nbrs, cnts, locs = [], [], []
    if with_blocks:
        nb = cb = 0
        for k, f in enumerate(fan.tolist()):
            nk = int(sizes[k])
            nbrs.append(nbr[nb:nb + nk * f].reshape(nk, f).copy())
            locs.append(loc[nb:nb + nk * f].reshape(nk, f).copy())
            cnts.append(cnt[cb:cb + nk].copy())
            nb += nk * f
            cb += nk
    return SampleResult(U[:n].copy(), sizes, nbrs, cnts, locs)


def gather(table: np.ndarray, row_bytes: int, idx) -> tuple:
    """out[r] = table[idx[r]] (bytes).  ``table`` is a flat uint8 array.  Returns (out, n_bad)."""
    table = np.ascontiguousarray(table).view(np.uint8).reshape(-1)
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64))
    rows = table.shape[0] // row_bytes
    n = idx.shape[0]
    out = np.zeros(n * row_bytes, dtype=np.uint8)
    bad = _L().oracle_gather(_p(table), rows, row_bytes, _p(idx) if n else None, n, _p(out))
    return out.reshape(n, row_bytes), int(bad)


def gather_into(table_addr: int, rows: int, row_bytes: int, idx: np.ndarray, out: np.ndarray) -> int:
    """Gather from a raw host table address (e.g. the registered shared mapping)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    return int(_L().oracle_gather(table_addr, rows, row_bytes, _p(idx), idx.shape[0], _p(out)))


def sample_and_gather(off, col, seeds, fanouts, rng_seed, table_addr, rows, row_bytes, out=None):
    """One minibatch fetch as the CPU oracle does it (used for the timed cpu_baseline leg)."""
    s = sample_uniform(off, col, seeds, fanouts, rng_seed, with_blocks=False)
    n = s.U.shape[0]
    if out is None or out.shape[0] < n * row_bytes:
        out = np.empty(n * row_bytes, dtype=np.uint8)
    gather_into(table_addr, rows, row_bytes, s.U, out)
    return s, out


def sage_mean_linear(x: np.ndarray, local: np.ndarray, cnt: np.ndarray, w: np.ndarray) -> np.ndarray:
    """The consumer's layer, in fp64: Y = A_hat . H . W^T for the first n_dst = len(cnt)
    rows, the paper's GCN layer H^(l+1) = A H^(l) W^(l) without the output non-linearity,
    with A_hat the sampled block's row-normalised adjacency including the self edge (GraphSAGE mean
    aggregation over the sampled neighbours):
        A_hat[i, i] += 1 / (1 + cnt[i]),  A_hat[i, local[i, q]] += 1 / (1 + cnt[i])  for q < cnt[i].
    x: [n_src, dim] rows of the minibatch (frontier order), local: [n_dst, fanout] positions in x,
    cnt: [n_dst], w: [hidden, dim].  Written row by row: h_i = (x_i + sum_q x_local[i,q]) / (1 + cnt_i),
    then Y = H . W^T (a library matmul as the second step)."""
    x = np.asarray(x, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    cnt = np.asarray(cnt, dtype=np.int64)
    n_dst = cnt.shape[0]
    h = np.empty((n_dst, x.shape[1]), dtype=np.float64)
    for i in range(n_dst):
        s = x[i].copy()
        for q in range(int(cnt[i])):
            s += x[int(local[i, q])]
        h[i] = s / (1.0 + cnt[i])
    return h @ w.T
