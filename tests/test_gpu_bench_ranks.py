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
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["ranks"] == 2     # kept at N > 1
    assert [r["rank"] for r in d["per_rank"]] == [0, 1] and all(r["register_s"] >= 0 for r in d["per_rank"])
    assert d["roofline"]["aggregate"]["achieved"] == d["value"]


def _run(extra, nproc=2, timeout=900):
    env = dict(os.environ, DGZ_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc), "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", str(nproc)] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return lines[0]


@pytest.mark.gpu
def test_bench_config5_two_ranks_one_gpu():
    """Config 5 under torchrun: fp16 rows of an odd dim (66 B, 2-byte aligned) at base offset 4 of a
    shared host buffer; every row of rank 0's last step equals the oracle's."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "5", "--row-bytes", "66", "--dtype", "f16", "--base", "4", "--table-gb", "2",
              "--steps", "4", "--warmup", "3", "--oracle-budget", "2"])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["parity"]["exact"] and d["parity"]["rows"] == d["config"]["rows_per_step"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["dma_baseline"]["ranks"] == 2 and d["e2e"]["value"] > 0
    assert d["config"]["row_bytes"] == 66 and len(d["per_rank"]) == 2


@pytest.mark.gpu
def test_bench_cache_two_ranks_one_gpu():
    """--cache-frac under torchrun: the hot rows sharded over 2 ranks (IPC-mapped shards), exact
    parity of rank 0's last minibatches, hit statistics and PCIe bytes avoided per rank."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "1", "--cache-frac", "0.2", "--steps", "5", "--warmup", "3", "--no-overlap",
              "--oracle-budget", "1"])
    assert d["parity"]["exact"] and d["config"]["cache"]["shards"] == 2
    cs = d["cache_stats"]
    assert 0 < cs["hit_rate_rank"] <= 1 and 0 < cs["peer_hit_rate_rank"] < cs["hit_rate_rank"]
    assert all(r["pcie_bytes_avoided"] > 0 for r in d["per_rank"])
