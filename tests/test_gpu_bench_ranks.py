"""bench.py under torchrun with 2 ranks sharing one GPU (DGZ_BENCH_SAME_DEVICE=1, gloo): the N > 1
code path -- shared /dev/shm table registered by every rank, seed partition j = i*G + rank,
max-over-ranks timing, all-rank DMA baseline, rank-0 oracle parity -- end to end."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_bench_two_ranks_one_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DGZ_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "1",
           "--steps", "5", "--warmup", "3", "--no-overlap"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                      # rank 0 prints one JSON line
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity"]["exact"]
    assert d["dma_baseline"]["ranks"] == 2
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
