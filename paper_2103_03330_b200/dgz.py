"""Thin Python binding of libdgz (include/dgz.h): argument marshalling only.

Every step of the hot path runs in libdgz's CUDA kernels; PyTorch supplies device memory,
pinned host buffers and streams.  There is no CPU or PyTorch fallback: if ``libdgz.so`` is
missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libdgz.so")

if not os.path.exists(_SO):
    raise ImportError(f"{_SO} is missing: build it with `python -m paper_2103_03330_b200.build` "
                      "(no CPU fallback exists by design)")

_lib = ctypes.CDLL(_SO)

# --- constants (dgz.h) -------------------------------------------------------------------------
OK, ERR_INVALID, ERR_CUDA, ERR_NOMEM, ERR_RANGE, ERR_STATE = range(6)
F32, F16, BF16, U8 = range(4)
REG_PORTABLE, REG_READONLY, REG_NO_PIN, REG_VMM_BACKED, REG_DEVICE, REG_MANAGED = 1, 2, 4, 8, 16, 32
HOST_HUGEPAGE, HOST_POPULATE, HOST_VMM, HOST_CUDA_PINNED, HOST_HUGETLB_2M, HOST_HUGETLB_1G = 1, 2, 4, 8, 16, 32
HOST_NUMA_INTERLEAVE = 64
HOST_MANAGED = 128
GATHER_AUTO, GATHER_SEGMENT, GATHER_NAIVE, GATHER_SHIFT, GATHER_BULK = range(5)
SCHED_AUTO, SCHED_INTERLEAVED, SCHED_BLOCKED = range(3)
FLAG_NO_MERGE, FLAG_DEEP, FLAG_ORDER, FLAG_STREAM_STORES, FLAG_EVICT_FIRST_LOADS, FLAG_DYNAMIC = 1, 2, 4, 8, 16, 32
MAX_FANOUT, MAX_LAYERS = 64, 8
ELEM_BYTES = {F32: 4, F16: 2, BF16: 2, U8: 1}
TORCH_DTYPE = {F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16, U8: torch.uint8}

_STATUS = {0: "OK", 1: "INVALID", 2: "CUDA", 3: "NOMEM", 4: "RANGE", 5: "STATE"}


class DgzError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: DGZ_ERR_{_STATUS.get(status, status)}: {last_error()}")


class RangeError(DgzError, IndexError):
    pass


def _check(st: int, where: str) -> None:
    if st != OK:
        raise (RangeError if st == ERR_RANGE else DgzError)(st, where)


# --- structs -----------------------------------------------------------------------------------
class TableInfo(ctypes.Structure):
    _fields_ = [("dev_ptr", ctypes.c_void_p), ("rows", ctypes.c_int64), ("dim", ctypes.c_int64),
                ("row_bytes", ctypes.c_int64), ("elem_bytes", ctypes.c_int32), ("device", ctypes.c_int32),
                ("base_mod128", ctypes.c_int32), ("flags", ctypes.c_int32), ("pinned_bytes", ctypes.c_int64),
                ("gpu_mem_delta", ctypes.c_int64), ("register_seconds", ctypes.c_double)]


class GatherCfg(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("sm_count", ctypes.c_int32), ("warps_per_cta", ctypes.c_int32),
                ("ctas_per_sm", ctypes.c_int32), ("schedule", ctypes.c_int32), ("flags", ctypes.c_int32)]


MAX_CACHE_SHARDS = 8


class CacheView(ctypes.Structure):
    _fields_ = [("slot_map", ctypes.c_void_p), ("n_shards", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("shards", ctypes.c_void_p * MAX_CACHE_SHARDS)]


class IpcHandle(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_ubyte * 64)]


class Csr(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("offsets", ctypes.c_void_p), ("cols", ctypes.c_void_p),
                ("cols_is64", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class SampleOut(ctypes.Structure):
    _fields_ = [("ids", ctypes.c_void_p), ("ids_cap", ctypes.c_int64), ("sizes_dev", ctypes.c_void_p),
                ("sizes_host", ctypes.c_void_p), ("nbr", ctypes.c_void_p), ("nbr_local", ctypes.c_void_p),
                ("cnt", ctypes.c_void_p), ("blocks_cap", ctypes.c_int64), ("cnt_cap", ctypes.c_int64),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("ids_sorted", ctypes.c_void_p), ("ids_sorted_pos", ctypes.c_void_p), ("rng_seed_dev", ctypes.c_void_p)]


_vp, _i64, _i32, _u64, _u32, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                    ctypes.c_uint32, ctypes.c_size_t)
_P = ctypes.POINTER

_SIGS = {
    "dgz_abi_version": ([], ctypes.c_int),
    "dgz_last_error": ([], ctypes.c_char_p),
    "dgz_device_sm_count": ([], ctypes.c_int),
    "dgz_kernel_launches": ([], ctypes.c_uint64),
    "dgz_host_numa_nodes": ([], ctypes.c_int),
    "dgz_host_alloc": ([ctypes.c_char_p, _sz, ctypes.c_int, _u32, _P(_vp)], ctypes.c_int),
    "dgz_host_free": ([_vp, _sz], ctypes.c_int),
    "dgz_host_unlink": ([ctypes.c_char_p], ctypes.c_int),
    "dgz_host_export": ([_vp, _P(ctypes.c_int)], ctypes.c_int),
    "dgz_host_import": ([ctypes.c_int, _sz, _P(_vp)], ctypes.c_int),
    "dgz_register_table": ([_vp, _i64, _i64, ctypes.c_int, _u32, _P(_vp)], ctypes.c_int),
    "dgz_unregister_table": ([_vp], ctypes.c_int),
    "dgz_wrap_device_table": ([_vp, _i64, _i64, ctypes.c_int, _P(_vp)], ctypes.c_int),
    "dgz_cache_fill": ([_vp, _vp, _i64, _P(CacheView), _vp], ctypes.c_int),
    "dgz_gather_cached": ([_vp, _P(CacheView), _vp, _vp, _i64, _vp, _vp, _P(GatherCfg), _vp], ctypes.c_int),
    "dgz_cache_fill_local": ([_vp, _vp, _i64, _P(CacheView), _i32, _vp], ctypes.c_int),
    "dgz_device_alloc": ([_sz, _P(_vp)], ctypes.c_int),
    "dgz_device_free": ([_vp], ctypes.c_int),
    "dgz_ipc_get_handle": ([_vp, _P(IpcHandle)], ctypes.c_int),
    "dgz_ipc_open": ([_P(IpcHandle), _P(_vp)], ctypes.c_int),
    "dgz_ipc_close": ([_vp], ctypes.c_int),
    "dgz_table_get_info": ([_vp, _P(TableInfo)], ctypes.c_int),
    "dgz_gather": ([_vp, _vp, _i64, _vp, _vp], ctypes.c_int),
    "dgz_gather_i32": ([_vp, _vp, _i64, _vp, _vp], ctypes.c_int),
    "dgz_gather_ex": ([_vp, _vp, _i64, _vp, _vp, _P(GatherCfg), _vp], ctypes.c_int),
    "dgz_gather_perm": ([_vp, _vp, _vp, _i64, _vp, _vp, _P(GatherCfg), _vp], ctypes.c_int),
    "dgz_gather_plan": ([_vp, _i64, _i32, _P(GatherCfg), _P(GatherCfg), _P(_i32)], ctypes.c_int),
    "dgz_order_workspace_bytes": ([_i64, _P(_sz)], ctypes.c_int),
    "dgz_order_ids": ([_vp, _i64, _i64, _vp, _vp, _vp, _sz, _vp], ctypes.c_int),
    "dgz_check_errors": ([_vp, _vp], ctypes.c_int),
    "dgz_sample_bounds": ([_i64, _i64, _P(_i32), ctypes.c_int, _P(_i64), _P(_i64), _P(_i64)], ctypes.c_int),
    "dgz_sample_workspace_bytes": ([_i64, _i64, _P(_sz)], ctypes.c_int),
    "dgz_sample_uniform": ([_P(Csr), _vp, _i64, _P(_i32), ctypes.c_int, _u64, _P(SampleOut), _vp], ctypes.c_int),
    "dgz_sample_check": ([_P(SampleOut), _vp], ctypes.c_int),
    "dgz_aggregate_mean": ([_vp, _i64, _vp, _vp, _i32, _vp, _i64, _vp, _i32, _i32, _i32, _vp], ctypes.c_int),
    "dgz_sage_mean_linear": ([_vp, _i64, _vp, _vp, _i32, _vp, _i64, _vp, _i64, _vp, _i32, _i32, _i32, _vp], ctypes.c_int),
    "dgz_sage_workspace": ([_i64, _i64, _P(_i64), _P(_i32)], ctypes.c_int),
    "dgz_partition_create": ([_i32, _i32, _u32, _P(_vp)], ctypes.c_int),
    "dgz_partition_get": ([_vp, _P(_vp), _P(_vp), _P(_i32), _P(_i32)], ctypes.c_int),
    "dgz_partition_group_count": ([_P(_i32), _P(_i32)], ctypes.c_int),
    "dgz_partition_create_groups": ([_P(_i32), _i32, _i32, _P(_vp)], ctypes.c_int),
    "dgz_partition_destroy": ([_vp], ctypes.c_int),
    "dgz_partition_stream": ([_vp, _i32, _i32, _P(_vp)], ctypes.c_int),
    "dgz_probe_stream": ([_vp, _i64, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "dgz_probe_chase": ([_vp, _i64, _vp, _vp], ctypes.c_int),
    "dgz_probe_stream_hint": ([_vp, _i64, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "dgz_probe_spin": ([_i32, _i32, _i64, _vp, _vp], ctypes.c_int),
    "dgz_probe_rows": ([_vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTS = tuple(_SIGS)


def abi_version() -> int:
    return _lib.dgz_abi_version()


def last_error() -> str:
    m = _lib.dgz_last_error()
    return m.decode() if m else ""


def device_sm_count() -> int:
    return _lib.dgz_device_sm_count()


def kernel_launches() -> int:
    return int(_lib.dgz_kernel_launches())


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _dptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return t.data_ptr()


# --- host table manager ------------------------------------------------------------------------
class HostBuffer:
    """Host mapping from dgz_host_alloc (anonymous or /dev/shm shared)."""

    def __init__(self, nbytes: int, shm_name: str | None = None, create: bool = True, flags: int = HOST_HUGEPAGE,
                 import_fd: int | None = None):
        p = _vp()
        if import_fd is not None:
            _check(_lib.dgz_host_import(import_fd, nbytes, ctypes.byref(p)), "dgz_host_import")
        else:
            name = shm_name.encode() if shm_name else None
            _check(_lib.dgz_host_alloc(name, nbytes, int(create), flags, ctypes.byref(p)), "dgz_host_alloc")
        self.ptr = p.value
        self.nbytes = nbytes
        self.shm_name = shm_name

    def export_fd(self) -> int:
        fd = ctypes.c_int(-1)
        _check(_lib.dgz_host_export(self.ptr, ctypes.byref(fd)), "dgz_host_export")
        return fd.value

    def numpy(self, offset: int = 0, nbytes: int | None = None):
        import numpy as np
        n = self.nbytes - offset if nbytes is None else nbytes
        buf = (ctypes.c_uint8 * n).from_address(self.ptr + offset)
        return np.frombuffer(buf, dtype=np.uint8)

    def free(self) -> None:
        if self.ptr:
            _check(_lib.dgz_host_free(self.ptr, self.nbytes), "dgz_host_free")
            self.ptr = 0

    def unlink(self) -> None:
        if self.shm_name:
            _check(_lib.dgz_host_unlink(self.shm_name.encode()), "dgz_host_unlink")


def host_numa_nodes() -> int:
    """Online NUMA nodes of the host (dgz_host_numa_nodes)."""
    return int(_lib.dgz_host_numa_nodes())


def host_unlink(shm_name: str) -> None:
    _check(_lib.dgz_host_unlink(shm_name.encode()), "dgz_host_unlink")


# --- table registration ------------------------------------------------------------------------
class Table:
    """A registered (pinned + mapped) host feature table: the paper's unified tensor."""

    def __init__(self, host_ptr: int, rows: int, dim: int, dtype: int = F32, flags: int = 0):
        h = _vp()
        _check(_lib.dgz_register_table(host_ptr, rows, dim, dtype, flags, ctypes.byref(h)), "dgz_register_table")
        self.handle = h.value
        self.dtype = dtype
        self.info = self.get_info()

    def get_info(self) -> TableInfo:
        info = TableInfo()
        _check(_lib.dgz_table_get_info(self.handle, ctypes.byref(info)), "dgz_table_get_info")
        return info

    @property
    def rows(self) -> int:
        return self.info.rows

    @property
    def row_bytes(self) -> int:
        return self.info.row_bytes

    def unregister(self) -> None:
        if self.handle:
            h, self.handle = self.handle, None      # the C handle is freed even when the call reports an error
            _check(_lib.dgz_unregister_table(h), "dgz_unregister_table")

    def __del__(self):
        try:
            self.unregister()
        except Exception:
            pass


def register_table(host_ptr: int, rows: int, dim: int, dtype: int = F32, flags: int = 0) -> Table:
    return Table(host_ptr, rows, dim, dtype, flags)


class DeviceTable(Table):
    """A table resident in HBM (dgz_wrap_device_table): the All-in-GPU reference."""

    def __init__(self, dev_ptr: int, rows: int, dim: int, dtype: int = F32):
        h = _vp()
        _check(_lib.dgz_wrap_device_table(dev_ptr, rows, dim, dtype, ctypes.byref(h)), "dgz_wrap_device_table")
        self.handle = h.value
        self.dtype = dtype
        self.info = self.get_info()


class HotRowCache:
    """Row-granular HBM cache of a registered table (dgz_cache_fill / dgz_gather_cached).
    Shards are local device memory here; peer-mapped shards use the same view (NVLink loads)."""

    def __init__(self, table: Table, hot_ids: torch.Tensor, n_shards: int = 1, stream=None):
        assert hot_ids.dtype == torch.int64 and hot_ids.is_cuda and 1 <= n_shards <= MAX_CACHE_SHARDS
        self.table = table
        n_hot = hot_ids.numel()
        per = (n_hot + n_shards - 1) // n_shards
        self.slot_map = torch.empty(table.rows, dtype=torch.int32, device=hot_ids.device)
        self.shards = [torch.empty((max(per, 1), table.row_bytes), dtype=torch.uint8, device=hot_ids.device)
                       for _ in range(n_shards)]
        self.view = CacheView(self.slot_map.data_ptr(), n_shards, 0)
        for g, sh in enumerate(self.shards):
            self.view.shards[g] = sh.data_ptr()
        self.n_hot = n_hot
        _check(_lib.dgz_cache_fill(table.handle, _dptr(hot_ids) if n_hot else None, n_hot, ctypes.byref(self.view),
                                   _stream(stream)), "dgz_cache_fill")

    def gather(self, idx: torch.Tensor, out: torch.Tensor, dst_pos: torch.Tensor | None = None, n: int | None = None,
               n_dev: torch.Tensor | None = None, cfg: GatherCfg | None = None, stream=None) -> torch.Tensor:
        n = idx.numel() if n is None else n
        assert idx.dtype == torch.int64
        _check(_lib.dgz_gather_cached(self.table.handle, ctypes.byref(self.view), _dptr(idx), _dptr(dst_pos), n,
                                      _dptr(n_dev), _dptr(out), ctypes.byref(cfg) if cfg is not None else None,
                                      _stream(stream)), "dgz_gather_cached")
        return out


class ShardedHotRowCache:
    """HBM row cache sharded across the ranks of a process group (one process per GPU; SURVEY 8(e),
    8(f) NEXT-1): rank g owns shard g (hot rows g, g + G, ...) in its own HBM and fills it by
    zero-copy (dgz_cache_fill_local); the shards' CUDA IPC handles are exchanged once with an
    object all-gather (setup, off the data path) and every rank maps the others' shards
    (dgz_ipc_open: NVLink peer memory on an 8-GPU box, the same HBM when ranks share a GPU).  The
    cached gather then reads each row from whichever GPU holds it, the rest over PCIe.  `group` is
    a torch.distributed process group (None = default)."""

    def __init__(self, table: Table, hot_ids: torch.Tensor, group=None, stream=None):
        import torch.distributed as dist
        assert hot_ids.dtype == torch.int64 and hot_ids.is_cuda
        G, g = dist.get_world_size(group), dist.get_rank(group)
        assert 1 <= G <= MAX_CACHE_SHARDS
        self.table, self.G, self.rank = table, G, g
        n_hot = hot_ids.numel()
        per = max((n_hot + G - 1) // G, 1)
        p = _vp()
        _check(_lib.dgz_device_alloc(per * table.row_bytes, ctypes.byref(p)), "dgz_device_alloc")
        self.local = p.value
        self.opened = []
        self.group = group
        self.slot_map = torch.empty(table.rows, dtype=torch.int32, device=hot_ids.device)
        self.view = CacheView(self.slot_map.data_ptr(), G, 0)
        self.view.shards[g] = self.local
        h = IpcHandle()
        try:
            _check(_lib.dgz_cache_fill_local(table.handle, _dptr(hot_ids) if n_hot else None, n_hot, ctypes.byref(self.view),
                                             g, _stream(stream)), "dgz_cache_fill_local")
            (torch.cuda.current_stream() if stream is None else stream).synchronize()
            _check(_lib.dgz_ipc_get_handle(self.local, ctypes.byref(h)), "dgz_ipc_get_handle")
        except Exception:
            _lib.dgz_device_free(self.local)
            self.local = None
            raise
        handles = [None] * G
        dist.all_gather_object(handles, bytes(h.bytes), group=group)   # also orders every fill before use
        for r, hb in enumerate(handles):
            if r == g:
                continue
            hr = IpcHandle()
            ctypes.memmove(hr.bytes, hb, 64)
            q = _vp()
            _check(_lib.dgz_ipc_open(ctypes.byref(hr), ctypes.byref(q)), "dgz_ipc_open")
            self.view.shards[r] = q.value
            self.opened.append(q.value)
        self.n_hot = n_hot

    def gather(self, idx: torch.Tensor, out: torch.Tensor, dst_pos: torch.Tensor | None = None, n: int | None = None,
               n_dev: torch.Tensor | None = None, cfg: GatherCfg | None = None, stream=None) -> torch.Tensor:
        n = idx.numel() if n is None else n
        assert idx.dtype == torch.int64
        assert self.local is not None, "ShardedHotRowCache is closed"
        _check(_lib.dgz_gather_cached(self.table.handle, ctypes.byref(self.view), _dptr(idx), _dptr(dst_pos), n,
                                      _dptr(n_dev), _dptr(out), ctypes.byref(cfg) if cfg is not None else None,
                                      _stream(stream)), "dgz_gather_cached")
        return out

    def close(self) -> None:
        """Collective: unmap the peers' shards, then (after every rank has) free this rank's shard."""
        import torch.distributed as dist
        torch.cuda.synchronize()
        for q in self.opened:
            _check(_lib.dgz_ipc_close(q), "dgz_ipc_close")
        self.opened = []
        dist.barrier(group=self.group)
        if self.local:
            _check(_lib.dgz_device_free(self.local), "dgz_device_free")
            self.local = None


def unregister_table(t: Table) -> None:
    t.unregister()


# --- gather ------------------------------------------------------------------------------------
def gather_cfg(variant: int = GATHER_AUTO, sm_count: int = 0, warps_per_cta: int = 0, ctas_per_sm: int = 0,
               schedule: int = SCHED_AUTO, flags: int = 0) -> GatherCfg:
    return GatherCfg(variant, sm_count, warps_per_cta, ctas_per_sm, schedule, flags)


VARIANT_NAMES = {GATHER_SEGMENT: "segment", GATHER_NAIVE: "naive", GATHER_SHIFT: "shift", GATHER_BULK: "bulk"}


def gather_plan(table: Table, n: int, sorted_ids: bool = True, cfg: GatherCfg | None = None) -> dict:
    """The launch a gather of n rows would use (dgz_gather_plan): variant, SMs, warps per CTA, CTAs,
    line loads in flight per lane, schedule, flags."""
    plan, ctas = GatherCfg(), _i32()
    _check(_lib.dgz_gather_plan(table.handle, int(n), int(bool(sorted_ids)), ctypes.byref(cfg) if cfg is not None else None,
                                ctypes.byref(plan), ctypes.byref(ctas)), "dgz_gather_plan")
    return {"variant": VARIANT_NAMES.get(plan.variant, plan.variant), "sm_count": plan.sm_count,
            "warps_per_cta": plan.warps_per_cta, "ctas": ctas.value,
            "line_loads_per_lane": 16 if plan.flags & FLAG_DEEP else 8,
            "schedule": ("work counter" if plan.flags & FLAG_DYNAMIC else
                         ("blocked" if plan.schedule == SCHED_BLOCKED else "static interleave")),
            "flags": plan.flags}


def gather(table: Table, idx: torch.Tensor, out: torch.Tensor, n: int | None = None, n_dev: torch.Tensor | None = None,
           cfg: GatherCfg | None = None, stream=None) -> torch.Tensor:
    """out[r] = table[idx[r]] for r < n (or < min(n, *n_dev)); asynchronous on ``stream``."""
    n = idx.numel() if n is None else n
    assert out.numel() * out.element_size() >= n * table.row_bytes, "out too small"
    s = _stream(stream)
    if idx.dtype == torch.int32 and n_dev is None and cfg is None:
        _check(_lib.dgz_gather_i32(table.handle, _dptr(idx), n, _dptr(out), s), "dgz_gather_i32")
        return out
    assert idx.dtype == torch.int64, "idx must be int64 (or int32 with the default config)"
    if n_dev is None and cfg is None:
        _check(_lib.dgz_gather(table.handle, _dptr(idx), n, _dptr(out), s), "dgz_gather")
    else:
        _check(_lib.dgz_gather_ex(table.handle, _dptr(idx), n, _dptr(n_dev), _dptr(out),
                                  ctypes.byref(cfg) if cfg is not None else None, s), "dgz_gather_ex")
    return out


def gather_perm(table: Table, idx: torch.Tensor, dst_pos: torch.Tensor, out: torch.Tensor, n: int | None = None,
                n_dev: torch.Tensor | None = None, cfg: GatherCfg | None = None, stream=None) -> torch.Tensor:
    """out[dst_pos[k]] = table[idx[k]] (dgz_gather_perm): fetch in table order, scatter to HBM."""
    n = idx.numel() if n is None else n
    assert idx.dtype == torch.int64 and dst_pos.dtype == torch.int64
    assert out.numel() * out.element_size() >= n * table.row_bytes, "out too small"
    _check(_lib.dgz_gather_perm(table.handle, _dptr(idx), _dptr(dst_pos), n, _dptr(n_dev), _dptr(out),
                                ctypes.byref(cfg) if cfg is not None else None, _stream(stream)), "dgz_gather_perm")
    return out


def order_ids(ids: torch.Tensor, max_id: int, stream=None) -> tuple:
    """(ids_sorted, pos) for dgz_gather_perm (dgz_order_ids); allocates outputs and workspace."""
    assert ids.dtype == torch.int64 and ids.is_cuda
    n = ids.numel()
    v = _sz()
    _check(_lib.dgz_order_workspace_bytes(n, ctypes.byref(v)), "dgz_order_workspace_bytes")
    ws = torch.empty(max(v.value, 1), dtype=torch.uint8, device=ids.device)
    srt = torch.empty_like(ids)
    pos = torch.empty_like(ids)
    _check(_lib.dgz_order_ids(_dptr(ids), n, max_id, _dptr(srt), _dptr(pos), ws.data_ptr(), v.value, _stream(stream)),
           "dgz_order_ids")
    return srt, pos


class Orderer:
    """dgz_order_ids with outputs and workspace allocated once for lists of up to ``max_n`` IDs
    (for loops that order a fresh list every step without allocating)."""

    def __init__(self, max_n: int, device=None):
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        v = _sz()
        _check(_lib.dgz_order_workspace_bytes(max_n, ctypes.byref(v)), "dgz_order_workspace_bytes")
        self.ws_bytes = v.value
        self.ws = torch.empty(max(v.value, 1), dtype=torch.uint8, device=device)
        self.srt = torch.empty(max(max_n, 1), dtype=torch.int64, device=device)
        self.pos = torch.empty(max(max_n, 1), dtype=torch.int64, device=device)
        self.max_n = max_n

    def order(self, ids: torch.Tensor, max_id: int, n: int | None = None, stream=None) -> tuple:
        n = ids.numel() if n is None else n
        assert ids.dtype == torch.int64 and ids.is_cuda and n <= self.max_n
        _check(_lib.dgz_order_ids(_dptr(ids), n, max_id, self.srt.data_ptr(), self.pos.data_ptr(), self.ws.data_ptr(),
                                  self.ws_bytes, _stream(stream)), "dgz_order_ids")
        return self.srt[:n], self.pos[:n]


def check_errors(table: Table, stream=None) -> None:
    _check(_lib.dgz_check_errors(table.handle, _stream(stream)), "dgz_check_errors")


# --- sampler -----------------------------------------------------------------------------------
def _i32arr(xs):
    return (ctypes.c_int32 * max(len(xs), 1))(*xs)


def sample_bounds(n_nodes: int, n_seeds: int, fanouts) -> tuple:
    fan = _i32arr(list(fanouts))
    L = len(fanouts)
    b = (ctypes.c_int64 * (L + 1))()
    be, ce = _i64(), _i64()
    _check(_lib.dgz_sample_bounds(n_nodes, n_seeds, fan, L, b, ctypes.byref(be), ctypes.byref(ce)), "dgz_sample_bounds")
    return list(b), be.value, ce.value


def sample_workspace_bytes(n_nodes: int, max_seeds: int) -> int:
    v = _sz()
    _check(_lib.dgz_sample_workspace_bytes(n_nodes, max_seeds, ctypes.byref(v)), "dgz_sample_workspace_bytes")
    return v.value


class SampleBuffers:
    """Caller-owned outputs + workspace of dgz_sample_uniform, sized by dgz_sample_bounds."""

    def __init__(self, n_nodes: int, max_seeds: int, fanouts, device=None, blocks: bool = True, local: bool = True,
                 sorted_ids: bool = True, device_rng: bool = False):
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else device
        self.fanouts = tuple(int(f) for f in fanouts)
        self.bounds, be, ce = sample_bounds(n_nodes, max_seeds, self.fanouts)
        L = len(self.fanouts)
        self.ids = torch.empty(max(self.bounds[-1], 1), dtype=torch.int64, device=device)
        self.sizes_dev = torch.zeros(L + 1, dtype=torch.int64, device=device)
        self.sizes_host = torch.zeros(L + 1, dtype=torch.int64).pin_memory()
        self.nbr = torch.empty(max(be, 1), dtype=torch.int64, device=device) if blocks else None
        self.cnt = torch.empty(max(ce, 1), dtype=torch.int32, device=device) if blocks else None
        self.local = torch.empty(max(be, 1), dtype=torch.int32, device=device) if (blocks and local) else None
        self.ids_sorted = torch.empty_like(self.ids) if sorted_ids else None
        self.ids_sorted_pos = torch.empty_like(self.ids) if sorted_ids else None
        wsb = sample_workspace_bytes(n_nodes, max_seeds)
        self.workspace = torch.empty(wsb, dtype=torch.uint8, device=device)
        self.rng_dev = torch.zeros(1, dtype=torch.int64, device=device) if device_rng else None
        self.struct = SampleOut(self.ids.data_ptr(), self.ids.numel(), self.sizes_dev.data_ptr(), self.sizes_host.data_ptr(),
                                _dptr(self.nbr), _dptr(self.local), _dptr(self.cnt), be, ce,
                                self.workspace.data_ptr(), wsb, _dptr(self.ids_sorted), _dptr(self.ids_sorted_pos),
                                _dptr(self.rng_dev))

    def hop_blocks(self, sizes=None):
        """Per-hop (nbr [n_k x f_k], cnt [n_k], local [n_k x f_k]) views (after a sync)."""
        sizes = self.sizes_host.tolist() if sizes is None else sizes
        out, nb, cb = [], 0, 0
        for k, f in enumerate(self.fanouts):
            nk = sizes[k]
            out.append((self.nbr[nb:nb + nk * f].view(nk, f), self.cnt[cb:cb + nk],
                        self.local[nb:nb + nk * f].view(nk, f) if self.local is not None else None))
            nb += self.bounds[k] * f
            cb += self.bounds[k]
        return out


class Graph:
    """CSR in HBM (dgz_csr)."""

    def __init__(self, offsets: torch.Tensor, cols: torch.Tensor):
        assert offsets.dtype == torch.int64 and cols.dtype in (torch.int32, torch.int64)
        self.offsets, self.cols = offsets, cols
        self.n_nodes = offsets.numel() - 1
        self.struct = Csr(self.n_nodes, offsets.data_ptr(), cols.data_ptr(), int(cols.dtype == torch.int64), 0)


class HostGraph:
    """CSR left in pinned, mapped host memory and read by the sampler with zero-copy loads
    (a graph whose CSR does not fit HBM is sampled where it lies, the way the
    paper's unified tensor leaves features in host memory).  The column array (and with
    ``offsets_in_hbm=False`` the offsets too) is registered like a feature table (dgz_register_table
    as a byte table: pin + map) and the sampler is given the device pointers through the same
    dgz_csr -- no other change on the path.  By default the offsets (8 B per node, a small fraction
    of the columns) are copied to HBM, so the sampler's host page walks are for columns only.
    ``offsets`` / ``cols`` are host addresses (ints) of int64 [n_nodes + 1] and int32/int64
    [n_edges] arrays the caller keeps alive, or numpy arrays (copied into HostBuffers here; with
    ``managed=True`` into DGZ_HOST_MANAGED memory, which the GPU maps with 2 MiB pages)."""

    def __init__(self, offsets, cols, n_nodes: int | None = None, n_edges: int | None = None,
                 cols_is64: bool | None = None, flags: int = REG_READONLY, offsets_in_hbm: bool = True,
                 managed: bool = False):
        import numpy as np
        self._owned = []
        self._copy_flags = HOST_MANAGED if managed else HOST_HUGEPAGE   # numpy inputs: where the copies live
        self.offsets_dev = None
        if isinstance(offsets, np.ndarray):
            assert offsets.dtype == np.int64 and cols.dtype in (np.int32, np.int64)
            n_nodes, n_edges, cols_is64 = offsets.size - 1, cols.size, cols.dtype == np.int64
            if offsets_in_hbm:
                self.offsets_dev = torch.from_numpy(offsets).cuda()
                offsets = 0
            else:
                offsets = self._copy_in(offsets)
            cols = self._copy_in(cols) if cols.size else 0
        elif offsets_in_hbm:
            import numpy as np
            hv = (ctypes.c_int64 * (int(n_nodes) + 1)).from_address(int(offsets))
            self.offsets_dev = torch.from_numpy(np.frombuffer(hv, dtype=np.int64)).cuda()
        assert n_nodes is not None and n_edges is not None and cols_is64 is not None
        self.n_nodes, self.n_edges, self.cols_is64 = int(n_nodes), int(n_edges), bool(cols_is64)
        self.off_table = self.col_table = None
        try:
            # offsets (8 B per node) go to HBM by default -- the columns (8-16x larger on real
            # graphs) are what does not fit; the sampler then walks host pages only for columns
            if not offsets_in_hbm:
                self.off_table = register_table(int(offsets), (self.n_nodes + 1) * 8, 1, U8, flags)
            col_dev = 0
            if self.n_edges:
                self.col_table = register_table(int(cols), self.n_edges * (8 if cols_is64 else 4), 1, U8, flags)
                col_dev = self.col_table.info.dev_ptr
        except Exception:
            self.close()
            raise
        off_dev = self.offsets_dev.data_ptr() if self.offsets_dev is not None else self.off_table.info.dev_ptr
        self.struct = Csr(self.n_nodes, off_dev, col_dev, int(self.cols_is64), 0)

    def _copy_in(self, a) -> int:
        import numpy as np
        hb = HostBuffer(max(a.nbytes, 1), flags=self._copy_flags)
        np.copyto(hb.numpy(0, a.nbytes).view(a.dtype), a)
        self._owned.append(hb)
        return hb.ptr

    def close(self) -> None:
        for t in (self.col_table, self.off_table):
            if t is not None:
                t.unregister()
        self.col_table = self.off_table = None
        self.offsets_dev = None
        for hb in self._owned:
            hb.free()
        self._owned = []


def sample_uniform(graph: Graph, seeds: torch.Tensor, fanouts, rng_seed: int, bufs: SampleBuffers, stream=None) -> SampleBuffers:
    assert seeds.dtype == torch.int64
    fan = _i32arr(list(fanouts))
    _check(_lib.dgz_sample_uniform(ctypes.byref(graph.struct), _dptr(seeds), seeds.numel(), fan, len(fanouts),
                                   rng_seed & (2**64 - 1), ctypes.byref(bufs.struct), _stream(stream)),
           "dgz_sample_uniform")
    return bufs


def sample_check(bufs: SampleBuffers, stream=None) -> None:
    _check(_lib.dgz_sample_check(ctypes.byref(bufs.struct), _stream(stream)), "dgz_sample_check")


# --- SM partition (green contexts) ----------------------------------------------------------------
PARTITION_FINE, PARTITION_SPREAD = 1, 2


class Partition:
    """Fetch / compute SM groups with one stream each (dgz_partition_*); streams are exposed as
    torch.cuda.ExternalStream so PyTorch work can be queued on the compute group."""

    def __init__(self, fetch_sms: int, fetch_priority: int = -1, flags: int = 0, groups=None):
        h = _vp()
        if groups is not None:     # explicit SM groups (dgz_partition_create_groups)
            arr = (ctypes.c_int32 * len(groups))(*groups)
            _check(_lib.dgz_partition_create_groups(arr, len(groups), fetch_priority, ctypes.byref(h)),
                   "dgz_partition_create_groups")
        else:
            _check(_lib.dgz_partition_create(fetch_sms, fetch_priority, flags, ctypes.byref(h)), "dgz_partition_create")
        self.handle = h.value
        fs, cs, fn, cn = _vp(), _vp(), _i32(), _i32()
        _check(_lib.dgz_partition_get(self.handle, ctypes.byref(fs), ctypes.byref(cs), ctypes.byref(fn), ctypes.byref(cn)),
               "dgz_partition_get")
        self.fetch_sms, self.compute_sms = fn.value, cn.value
        self.fetch_stream = torch.cuda.ExternalStream(fs.value)
        self.compute_stream = torch.cuda.ExternalStream(cs.value)

    def stream(self, group: int = 0, priority: int = 0):
        """Another stream on the fetch (0) or compute (1) SMs, owned by the partition (dgz_partition_stream)."""
        st = _vp()
        _check(_lib.dgz_partition_stream(self.handle, group, priority, ctypes.byref(st)), "dgz_partition_stream")
        return torch.cuda.ExternalStream(st.value)

    def destroy(self) -> None:
        if self.handle:
            torch.cuda.synchronize()
            _check(_lib.dgz_partition_destroy(self.handle), "dgz_partition_destroy")
            self.handle = None


def partition_groups() -> tuple:
    """(number of minimal SM groups, SMs per group) of the current device (dgz_partition_group_count)."""
    n, per = _i32(), _i32()
    _check(_lib.dgz_partition_group_count(ctypes.byref(n), ctypes.byref(per)), "dgz_partition_group_count")
    return n.value, per.value


# --- stand-in consumer, probes -------------------------------------------------------------------
def aggregate_mean(x: torch.Tensor, dim: int, nbr_local: torch.Tensor, cnt: torch.Tensor, fanout: int,
                   n_dst_dev: torch.Tensor | None, n_dst_max: int, y: torch.Tensor, repeat: int = 1, sm_count: int = 0,
                   ctas_per_sm: int = 0, stream=None) -> torch.Tensor:
    _check(_lib.dgz_aggregate_mean(_dptr(x), dim, _dptr(nbr_local), _dptr(cnt), fanout, _dptr(n_dst_dev), n_dst_max,
                                   _dptr(y), repeat, sm_count, ctas_per_sm, _stream(stream)), "dgz_aggregate_mean")
    return y


def sage_mean_linear(x: torch.Tensor, dim: int, nbr_local: torch.Tensor, cnt: torch.Tensor, fanout: int,
                     n_dst_dev: torch.Tensor | None, n_dst_max: int, w: torch.Tensor, y: torch.Tensor, repeat: int = 1,
                     sm_count: int = 0, ctas_per_sm: int = 0, stream=None) -> torch.Tensor:
    """dgz_sage_mean_linear: y[:n_dst] = bf16(mean over self + sampled neighbours of x) @ w.T on the
    tensor cores; w is bf16 [hidden, dim], y fp32 [>= n_dst, hidden]."""
    assert w.dtype == torch.bfloat16 and w.dim() == 2 and w.shape[1] == dim, "w must be bf16 [hidden, dim]"
    _check(_lib.dgz_sage_mean_linear(_dptr(x), dim, _dptr(nbr_local), _dptr(cnt), fanout, _dptr(n_dst_dev), n_dst_max,
                                     _dptr(w), int(w.shape[0]), _dptr(y), repeat, sm_count, ctas_per_sm, _stream(stream)),
           "dgz_sage_mean_linear")
    return y


def sage_workspace(dim: int, hidden: int) -> tuple:
    """(shared-memory bytes, TMEM columns) of one dgz_sage_mean_linear CTA."""
    b, c = _i64(), _i32()
    _check(_lib.dgz_sage_workspace(dim, hidden, ctypes.byref(b), ctypes.byref(c)), "dgz_sage_workspace")
    return b.value, c.value


def probe_stream(src_dev_ptr: int, nbytes: int, sm_count: int, warps: int, unroll: int, sink: torch.Tensor, stream=None):
    _check(_lib.dgz_probe_stream(src_dev_ptr, nbytes, sm_count, warps, unroll, _dptr(sink), _stream(stream)),
           "dgz_probe_stream")


def probe_stream_hint(src_dev_ptr: int, nbytes: int, sm_count: int, warps: int, l2_prefetch_bytes: int, sink: torch.Tensor,
                      stream=None):
    _check(_lib.dgz_probe_stream_hint(src_dev_ptr, nbytes, sm_count, warps, l2_prefetch_bytes, _dptr(sink), _stream(stream)),
           "dgz_probe_stream_hint")


def probe_chase(src_dev_ptr: int, steps: int, cycles: torch.Tensor, stream=None):
    _check(_lib.dgz_probe_chase(src_dev_ptr, steps, _dptr(cycles), _stream(stream)), "dgz_probe_chase")


def probe_rows(src_dev_ptr: int, row_bytes: int, ids: torch.Tensor, sm_count: int, warps: int, rows_in_flight: int,
               sink: torch.Tensor, stream=None):
    """dgz_probe_rows: read the rows ids of src (row_bytes each), nothing written (random-row read ceiling)."""
    _check(_lib.dgz_probe_rows(src_dev_ptr, row_bytes, _dptr(ids), ids.numel(), sm_count, warps, rows_in_flight, _dptr(sink),
                               _stream(stream)), "dgz_probe_rows")


def probe_spin(ctas: int, threads: int, iters: int, sink: torch.Tensor, stream=None):
    _check(_lib.dgz_probe_spin(ctas, threads, iters, _dptr(sink), _stream(stream)), "dgz_probe_spin")
