"""The C ABI library loads and exports every symbol include/dgz.h declares (no GPU needed)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2103_03330_b200", "libdgz.so")


def _declared():
    src = open(os.path.join(ROOT, "include", "dgz.h")).read()
    return sorted(set(re.findall(r"DGZ_API\s+[\w\s\*]+?\b(dgz_\w+)\s*\(", src)))


def _lib():
    if not os.path.exists(SO):
        from paper_2103_03330_b200 import build
        build.build()
    return ctypes.CDLL(SO)


def test_exports_every_declared_symbol():
    names = _declared()
    assert len(names) >= 20
    lib = _lib()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the binding wraps exactly the declared entry points
    from paper_2103_03330_b200 import dgz
    assert sorted(dgz.EXPORTS) == names


def test_host_only_entry_points():
    from paper_2103_03330_b200 import dgz
    assert dgz.abi_version() == 1
    b, be, ce = dgz.sample_bounds(111_059_956, 1024, (15, 10, 5))
    assert b == [1024, 16384, 180224, 1081344]          # 1,081,344 for config 4
    assert be == 1024 * 15 + 16384 * 10 + 180224 * 5 and ce == 1024 + 16384 + 180224
    assert dgz.sample_bounds(10, 1024, (15,))[0] == [10, 10]
    assert dgz.sample_workspace_bytes(111_059_956, 1024) > 111_059_956 // 8 * 2


def test_invalid_arguments_fail_synchronously():
    from paper_2103_03330_b200 import dgz
    lib = dgz._lib
    h = ctypes.c_void_p()
    assert lib.dgz_register_table(None, 10, 4, dgz.F32, 0, ctypes.byref(h)) == dgz.ERR_INVALID
    assert "null" in dgz.last_error()
    assert lib.dgz_register_table(ctypes.c_void_p(4096), 0, 4, dgz.F32, 0, ctypes.byref(h)) == dgz.ERR_INVALID
    assert lib.dgz_register_table(ctypes.c_void_p(4096), 1, 4, 9, 0, ctypes.byref(h)) == dgz.ERR_INVALID
    assert lib.dgz_gather(None, None, 5, None, None) == dgz.ERR_INVALID
    fan = (ctypes.c_int32 * 1)(65)
    assert lib.dgz_sample_bounds(10, 1, fan, 1, None, None, None) == dgz.ERR_INVALID


def test_host_table_manager_shared_mapping():
    from paper_2103_03330_b200 import dgz
    name = f"/dgz_abi_test_{os.getpid()}"
    a = dgz.HostBuffer(1 << 16, name, create=True)
    try:
        a.numpy()[:8] = list(range(8))
        b = dgz.HostBuffer(1 << 16, name, create=False)
        assert b.numpy()[:8].tolist() == list(range(8))
        assert a.ptr % 4096 == 0
        b.free()
    finally:
        a.unlink()
        a.free()


def test_numa_interleaved_host_allocation():
    """DGZ_HOST_NUMA_INTERLEAVE: anonymous and /dev/shm mappings are created (interleaved over the
    online nodes on a multi-socket host, unchanged on one node) and are ordinary memory."""
    import numpy as np
    from paper_2103_03330_b200 import dgz
    assert dgz.host_numa_nodes() >= 1
    a = dgz.HostBuffer(8 << 20, flags=dgz.HOST_NUMA_INTERLEAVE | dgz.HOST_HUGEPAGE)
    name = f"/dgz_numa_test_{os.getpid()}"
    b = dgz.HostBuffer(4 << 20, name, create=True, flags=dgz.HOST_NUMA_INTERLEAVE)
    try:
        for buf in (a, b):
            v = buf.numpy()
            v[::4096] = 7
            assert int(v[::4096].sum()) == 7 * v[::4096].size and int(v[1::4096].sum()) == 0
    finally:
        a.free()
        b.unlink()
        b.free()


def test_binding_constants_match_the_header():
    """Every flag the binding exposes has the value include/dgz.h defines (HOST_*, REG_*, FLAG_*)."""
    from paper_2103_03330_b200 import dgz
    src = open(os.path.join(ROOT, "include", "dgz.h")).read()
    defs = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define\s+DGZ_(\w+)\s+(\d+)u?\b", src)}
    pairs = {"HOST_HUGEPAGE": "HOST_HUGEPAGE", "HOST_POPULATE": "HOST_POPULATE", "HOST_VMM": "HOST_VMM",
             "HOST_CUDA_PINNED": "HOST_CUDA_PINNED", "HOST_HUGETLB_2M": "HOST_HUGETLB_2M",
             "HOST_HUGETLB_1G": "HOST_HUGETLB_1G", "HOST_NUMA_INTERLEAVE": "HOST_NUMA_INTERLEAVE",
             "HOST_MANAGED": "HOST_MANAGED", "REG_PORTABLE": "REG_PORTABLE", "REG_READONLY": "REG_READONLY",
             "REG_NO_PIN": "REG_NO_PIN", "REG_VMM_BACKED": "REG_VMM_BACKED", "REG_DEVICE": "REG_DEVICE",
             "REG_MANAGED": "REG_MANAGED", "GATHER_FLAG_NO_MERGE": "FLAG_NO_MERGE", "GATHER_FLAG_DEEP": "FLAG_DEEP",
             "GATHER_FLAG_ORDER": "FLAG_ORDER", "GATHER_FLAG_STREAM_STORES": "FLAG_STREAM_STORES",
             "GATHER_FLAG_EVICT_FIRST_LOADS": "FLAG_EVICT_FIRST_LOADS", "GATHER_FLAG_DYNAMIC": "FLAG_DYNAMIC"}
    for h, py in pairs.items():
        assert h in defs, h
        assert getattr(dgz, py) == defs[h], (h, defs[h], getattr(dgz, py))
    # flag bits of one family never collide
    for fam in ("HOST_", "REG_", "GATHER_FLAG_"):
        vals = [v for k, v in defs.items() if k.startswith(fam)]
        assert len(vals) == len(set(vals)), fam


def test_host_alloc_path_names(tmp_path):
    """dgz_host_alloc with a path instead of a /dev/shm name: a file (created and truncated here)
    and another process's memfd reached through /proc/<pid>/fd/<n> -- the bench's fallback when
    /dev/shm is too small for the shared table.  CPU only."""
    from paper_2103_03330_b200 import dgz
    path = str(tmp_path / "table.bin")
    a = dgz.HostBuffer(1 << 16, path, create=True, flags=0)
    try:
        a.numpy()[:8] = list(range(1, 9))
        b = dgz.HostBuffer(1 << 16, path, create=False, flags=0)
        assert list(b.numpy()[:8]) == list(range(1, 9))       # the same pages through a second mapping
        b.free()
        a.unlink()
        assert not os.path.exists(path)
    finally:
        a.free()
    fd = os.memfd_create("dgz_abi_memfd", 0)
    try:
        os.ftruncate(fd, 1 << 16)
        os.pwrite(fd, bytes([7, 7, 7]), 100)
        m = dgz.HostBuffer(1 << 16, f"/proc/{os.getpid()}/fd/{fd}", create=False, flags=0)
        assert list(m.numpy()[100:103]) == [7, 7, 7]
        m.numpy()[200] = 9
        assert os.pread(fd, 1, 200) == bytes([9])
        m.unlink()                                               # a no-op for /proc paths
        m.free()
    finally:
        os.close(fd)
