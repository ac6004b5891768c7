"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds none of the method's arithmetic (no sampling, no gather): it makes the
graph, the feature-table bytes, the per-batch seed lists and the per-batch sampler seeds
that both sides consume (SURVEY.md section 8(d) table
"Concrete synthetic inputs").  The heavy lifting is plain C + OpenMP in ``gen.c`` so that the
papers100M-shaped inputs (1.6e9 edges, 56.9 GB of features) generate in seconds.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_SO = os.path.join(_HERE, "libdgzgen.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c -> libdgzgen.so (gcc, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        i64, u64, vp, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_double
        L.dgz_gen_offsets.argtypes = [i64, dbl, u64, vp]
        L.dgz_gen_offsets.restype = i64
        L.dgz_gen_cols32.argtypes = [i64, i64, u64, vp]
        L.dgz_gen_cols64.argtypes = [i64, i64, u64, vp]
        L.dgz_gen_fill.argtypes = [vp, i64, u64]
        L.dgz_gen_fill_f32.argtypes = [vp, i64, u64]
        L.dgz_gen_batch_seeds.argtypes = [i64, i64, u64, i64, vp]
        L.dgz_gen_batch_seeds.restype = i64
        L.dgz_gen_batch_rng_seed.argtypes = [u64, i64]
        L.dgz_gen_batch_rng_seed.restype = u64
        L.dgz_gen_random_ids.argtypes = [i64, i64, u64, vp]
        L.dgz_gen_distinct_ids.argtypes = [i64, i64, u64, vp]
        L.dgz_gen_set_threads.argtypes = [ctypes.c_int]
        L.dgz_gen_cols32_skewed.argtypes = [i64, i64, u64, dbl, vp]
        _lib = L
    return _lib


def _ptr(a) -> int:
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return int(a)


def set_threads(n: int) -> None:
    """OpenMP threads of the generators (results do not depend on it)."""
    lib().dgz_gen_set_threads(int(n))


# ----------------------------------------------------------------------------------------------
# graph, table, seeds
# ----------------------------------------------------------------------------------------------

def gen_csr(n: int, avg_degree: float, seed: int, col_dtype=np.int32, skew_alpha: float = 0.0):
    """CSR with Poisson(avg_degree) out-degrees and uniform endpoints; with
    skew_alpha > 1 the endpoints are power-law skewed (hot-row cache experiments, NEXT-1)."""
    off = np.empty(n + 1, dtype=np.int64)
    e = lib().dgz_gen_offsets(n, float(avg_degree), seed, _ptr(off))
    if e < 0:
        raise ValueError("bad graph parameters")
    col = np.empty(e, dtype=col_dtype)
    if skew_alpha > 1.0:
        assert col_dtype == np.int32 and n < 2**31
        lib().dgz_gen_cols32_skewed(n, e, seed, float(skew_alpha), _ptr(col))
    elif col_dtype == np.int32:
        assert n < 2**31
        lib().dgz_gen_cols32(n, e, seed, _ptr(col))
    else:
        lib().dgz_gen_cols64(n, e, seed, _ptr(col))
    return off, col


def gen_csr_into(n: int, avg_degree: float, seed: int, alloc, skew_alpha: float = 0.0):
    """gen_csr (int32 columns) written into caller memory: ``alloc(nbytes)`` returns a writable
    address (e.g. a shared /dev/shm mapping one rank fills for all).  Returns (offsets address,
    cols address, n_edges); the bytes equal gen_csr's with the same skew_alpha."""
    assert n < 2**31
    po = int(alloc((n + 1) * 8))
    e = lib().dgz_gen_offsets(n, float(avg_degree), seed, po)
    if e < 0:
        raise ValueError("bad graph parameters")
    pc = int(alloc(max(e * 4, 1)))
    if skew_alpha > 1.0:
        lib().dgz_gen_cols32_skewed(n, e, seed, float(skew_alpha), pc)
    else:
        lib().dgz_gen_cols32(n, e, seed, pc)
    return po, pc, int(e)


def fill_table(buf, nbytes: int, seed: int) -> None:
    """Fill ``nbytes`` bytes at ``buf`` (numpy array or raw address) with keyed random bits."""
    lib().dgz_gen_fill(_ptr(buf), int(nbytes), seed)


def fill_table_f32(buf, count: int, seed: int) -> None:
    """Fill ``count`` fp32 values at ``buf`` (numpy array or raw address) with finite keyed values in
    [-1, 1) (multiples of 2^-23), in parallel."""
    lib().dgz_gen_fill_f32(_ptr(buf), int(count), seed)


def table_bytes(nbytes: int, seed: int) -> np.ndarray:
    a = np.empty(nbytes, dtype=np.uint8)
    fill_table(a, nbytes, seed)
    return a


def batch_seeds(n: int, batch: int, seed: int, j: int) -> np.ndarray:
    """Seeds of global batch j: a slice of the epoch permutation."""
    out = np.empty(batch, dtype=np.int64)
    c = lib().dgz_gen_batch_seeds(n, batch, seed, j, _ptr(out))
    return out[:c].copy()


def batch_rng_seed(seed: int, j: int) -> int:
    return int(lib().dgz_gen_batch_rng_seed(seed & (2**64 - 1), j))


def random_ids(rows: int, n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    lib().dgz_gen_random_ids(rows, n, seed, _ptr(out))
    return out


def distinct_ids(rows: int, n: int, seed: int) -> np.ndarray:
    assert n <= rows
    out = np.empty(n, dtype=np.int64)
    lib().dgz_gen_distinct_ids(rows, n, seed, _ptr(out))
    return out


def adjacent_run_ids(rows: int, n: int, seed: int, max_run: int = 8) -> np.ndarray:
    """n IDs made of runs of 1..max_run table-adjacent rows (start uniform), plus a few repeats,
    in shuffled run order: the dense lists whose sorted order puts neighbouring rows side by side
    (two rows sharing a 128 B line), as a dense minibatch does."""
    rng = np.random.default_rng(seed)
    parts, got = [], 0
    while got < n:
        k = int(rng.integers(1, max_run + 1))
        s = int(rng.integers(0, max(rows - k, 1)))
        run = np.arange(s, min(s + k, rows), dtype=np.int64)
        parts.append(run)
        got += run.shape[0]
    ids = np.concatenate(parts)[:n]
    if n > 16:   # duplicates
        j = rng.integers(0, n, size=max(1, n // 64))
        ids[rng.integers(0, n, size=j.shape[0])] = ids[j]
    return ids


def float_table(count: int, seed: int) -> np.ndarray:
    """count finite fp32 values, uniform in [-1, 1) (for consumers that do arithmetic on rows)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=count).astype(np.float32)


def rank_batches(rank: int, world: int, steps: int, start: int = 0):
    """Global batch indices owned by ``rank``: j = start + g*world + rank (j mod G == rank)."""
    return [start + i * world + rank for i in range(steps)]


# ----------------------------------------------------------------------------------------------
# workload configurations (BASELINE.json "configs")
# ----------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    cid: int
    name: str
    n_nodes: int
    avg_degree: float
    dim: int
    elem: int            # bytes per element (4 = fp32)
    fanouts: tuple
    batch: int
    base_seed: int = field(default=0)

    @property
    def row_bytes(self) -> int:
        return self.dim * self.elem

    @property
    def table_bytes(self) -> int:
        return self.n_nodes * self.row_bytes

    @property
    def seed(self) -> int:
        return 0x5EED + self.cid


CONFIGS = {
    1: Config(1, "tiny-10k", 10_000, 10.0, 128, 4, (10, 5), 1024),
    2: Config(2, "reddit-shaped", 233_000, 492.0, 602, 4, (25, 10), 1024),
    3: Config(3, "ogbn-products-shaped", 2_449_029, 50.5, 100, 4, (15, 10, 5), 1024),
    4: Config(4, "ogbn-papers100M-shaped", 111_059_956, 14.4, 128, 4, (15, 10, 5), 1024),
}

# config 5: row widths (bytes) of the fig:alignment_measurement-style sweep
SWEEP_ROW_BYTES = (16, 32, 48, 64, 96, 100, 128, 132, 200, 256, 260, 400, 480, 512, 516, 1024,
                   1028, 1032, 1036, 1040, 1044, 1260, 2048, 2312, 2408, 4096)
SWEEP_BASE_OFFSETS = (0, 4, 8, 16, 64)


def sample_bound(n_nodes: int, n_seeds: int, fanouts) -> list:
    """Upper bound on |F_k| for k = 0..L: min(N, n_seeds * prod_{i<k} (1 + f_i))."""
    out, b = [], n_seeds
    out.append(min(n_nodes, b))
    for f in fanouts:
        b = b * (1 + f)
        out.append(min(n_nodes, b))
    return out
