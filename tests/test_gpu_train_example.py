"""NEXT-4 example (examples/graphsage_train.py) runs end to end: GraphSAGE training fed by the
zero-copy fetcher, the CPU-gather + cudaMemcpy baseline and the All-in-GPU table, on one process
and under torchrun with DDP (2 ranks sharing one GPU, gloo)."""
import json
import math
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import dgz_inputs as gen
import oracle

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


def _oracle_anchor(path, with_blocks):
    """The minibatch the example's training consumed (dumped by --dump) equals the CPU oracle's: U,
    every gathered row (from the same config-1 table bytes), and the per-hop blocks the model reads."""
    c = gen.CONFIGS[1]
    z = np.load(path)
    j = int(z["j"])
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    want = oracle.sample_uniform(off, col, gen.batch_seeds(c.n_nodes, c.batch, c.seed, j), c.fanouts,
                                 gen.batch_rng_seed(c.seed, j))
    assert np.array_equal(z["U"], want.U)
    rows, bad = oracle.gather(gen.table_bytes(c.table_bytes, c.seed), c.row_bytes, want.U)
    assert bad == 0 and np.array_equal(z["rows"].reshape(rows.shape), rows)
    if with_blocks:
        for k in range(len(c.fanouts)):
            assert np.array_equal(z[f"cnt{k}"], want.cnt[k]) and np.array_equal(z[f"loc{k}"], want.local[k])


def test_train_example_single_process(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, EX, "--config", "1", "--steps", "3", "--fetch-sms", "8", "--dump", str(tmp_path)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _check(r.stdout, ("zc", "dma", "hbm"))
    assert math.isfinite(d["zc"]["loss"]) and d["zc"]["loss"] == d["hbm"]["loss"]   # same rows, same model
    assert d["speedup_zc_over_dma"] > 0
    _oracle_anchor(tmp_path / "zc_rank0.npz", True)      # what zero-copy training consumed = the oracle's
    _oracle_anchor(tmp_path / "dma_rank0.npz", False)    # and the DMA baseline moved the same bytes


def test_train_example_ddp_two_ranks(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, DGZ_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), EX, "--config", "1", "--steps", "3", "--fetch-sms", "8", "--modes", "zc,dma",
           "--dump", str(tmp_path)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    err = "\n".join(l for l in r.stderr.splitlines() if "rank0" in l or "Error" in l)
    assert r.returncode == 0, r.stdout[-2000:] + err[-4000:]
    d = _check(r.stdout, ("zc", "dma"))
    assert d["ranks"] == 2 and len(d["zc"]["per_rank"]) == 2
    for rank in (0, 1):                                  # each rank's minibatch (j = i*G + rank) vs the oracle
        _oracle_anchor(tmp_path / f"zc_rank{rank}.npz", True)
        _oracle_anchor(tmp_path / f"dma_rank{rank}.npz", False)
    assert int(np.load(tmp_path / "zc_rank1.npz")["j"]) == 1


def test_train_example_uvm_modes():
    """The UVM baselines (managed memory: migrated on fault / host-preferred and mapped) train on the
    same minibatches through the same fetcher; the losses equal the zero-copy run's (same rows)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, EX, "--config", "1", "--steps", "3", "--fetch-sms", "8", "--modes", "zc,uvm,uvm_host"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    d = _check(r.stdout, ("zc", "uvm", "uvm_host"))
    for m in ("uvm", "uvm_host"):
        assert d[m]["first_pass_fetch_ms"] > 0 and d[m]["loss"] == d["zc"]["loss"]
