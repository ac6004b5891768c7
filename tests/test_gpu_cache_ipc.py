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
