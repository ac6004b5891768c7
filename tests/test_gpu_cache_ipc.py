"""HBM row cache sharded across ranks: torchrun with 2 and 3 ranks on one
GPU (gloo); every rank owns one shard, maps the others' through CUDA IPC (the same calls map peer
GPUs' HBM over NVLink on a multi-GPU box) and its cached gathers must equal the oracle's."""
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ranks,R,base", [(2, 400, 0), (3, 2408, 8), (2, 100, 4)])
def test_sharded_cache_over_ipc(ranks, R, base):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, CACHE_R=str(R), CACHE_BASE=str(base))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks), "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "workers", "cache_ipc_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert sum(" ok: " in l for l in r.stdout.splitlines()) == ranks, r.stdout


def test_cache_and_ipc_argument_errors():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes
    sys.path.insert(0, ROOT)
    from paper_2103_03330_b200 import dgz
    torch.cuda.set_device(0)
    lib = dgz._lib
    p = ctypes.c_void_p()
    assert lib.dgz_device_alloc(0, ctypes.byref(p)) == dgz.ERR_INVALID
    h = dgz.IpcHandle()                                            # all-zero handle: not a real allocation
    assert lib.dgz_ipc_open(ctypes.byref(h), ctypes.byref(p)) == dgz.ERR_CUDA
    assert lib.dgz_ipc_close(None) == dgz.ERR_INVALID
    import dgz_inputs as gen
    buf = dgz.HostBuffer(1 << 20)
    gen.fill_table(buf.ptr, 1 << 20, 3)
    t = dgz.register_table(buf.ptr, 1024, 256, dgz.F32)
    try:
        hot = torch.arange(10, dtype=torch.int64, device="cuda")
        slot = torch.empty(1024, dtype=torch.int32, device="cuda")
        shard = torch.empty(10 * 1024, dtype=torch.uint8, device="cuda")
        view = dgz.CacheView(slot.data_ptr(), 2, 0)
        view.shards[0] = shard.data_ptr()                           # shard 1 left NULL: owned by another rank
        assert lib.dgz_cache_fill_local(t.handle, hot.data_ptr(), 10, ctypes.byref(view), 2, None) == dgz.ERR_INVALID
        assert lib.dgz_cache_fill(t.handle, hot.data_ptr(), 10, ctypes.byref(view), None) == dgz.ERR_INVALID
        assert lib.dgz_cache_fill_local(t.handle, hot.data_ptr(), 10, ctypes.byref(view), 0, None) == dgz.OK
        torch.cuda.synchronize()
        assert slot[:10].tolist() == list(range(10)) and int((slot[10:] == -1).sum()) == 1014
        want = torch.from_numpy(buf.numpy(0, 1024 * 1024)).view(1024, 1024)[0:10:2]
        assert torch.equal(shard.view(10, 1024)[:5].cpu(), want)   # shard 0 = hot rows 0, 2, 4, 6, 8
    finally:
        t.unregister()
        buf.free()
