"""NEXT-4 example (examples/graphsage_train.py) runs end to end: GraphSAGE training fed by the
zero-copy fetcher, the CPU-gather + cudaMemcpy baseline and the All-in-GPU table, on one process
and under torchrun with DDP (2 ranks sharing one GPU, gloo)."""
import json
import math
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EX = os.path.join(ROOT, "examples", "graphsage_train.py")
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check(out, modes):
    lines = [json.loads(l) for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    for m in modes:
        assert d[m]["step_ms"] > 0
    return d


def test_train_example_single_process():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, EX, "--config", "1", "--steps", "3", "--fetch-sms", "8"], capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _check(r.stdout, ("zc", "dma", "hbm"))
    assert math.isfinite(d["zc"]["loss"]) and d["zc"]["loss"] == d["hbm"]["loss"]   # same rows, same model
    assert d["speedup_zc_over_dma"] > 0


def test_train_example_ddp_two_ranks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DGZ_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), EX, "--config", "1", "--steps", "3", "--fetch-sms", "8", "--modes", "zc,dma"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    err = "\n".join(l for l in r.stderr.splitlines() if "rank0" in l or "Error" in l)
    assert r.returncode == 0, r.stdout[-2000:] + err[-4000:]
    d = _check(r.stdout, ("zc", "dma"))
    assert d["ranks"] == 2 and len(d["zc"]["per_rank"]) == 2
