"""bench.py host-side logic on CPU (no GPU): the N > 1 preflight (shared /dev/shm, RAM, memlock;
one rank's problem stops every rank), the shared power-law CSR of the --cache-frac mode, host-core
placement helpers, the workload label both arms print, and the overlap timeline writer."""
import argparse
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import dgz_inputs as gen  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_preflight_single_rank():
    d = bench.Dist(1)
    info = bench.preflight(d, 1 << 20, 1 << 20)
    assert info["mem_available_gb"] is None or info["mem_available_gb"] > 0
    with pytest.raises(bench.PreflightError, match="host RAM"):
        bench.preflight(d, 1 << 60, 0)


def _preflight_worker(rank, world, port, q):
    try:
        os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                           "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
        sys.path.insert(0, ROOT)
        import bench as b
        from paper_2103_03330_b200 import dgz
        d = b.Dist(world)
        ok_small = b.preflight(d, 1 << 20, 1 << 20)
        try:
            b.preflight(d, 1 << 60, 0)          # only rank 0 checks the shared objects ...
            raised = None
        except b.PreflightError as e:           # ... but every rank must stop
            raised = str(e)
        # the --cache-frac mode's power-law CSR, generated once into /dev/shm and mapped by all
        cfg = gen.CONFIGS[1]
        off, col, e, bufs = b.make_csr(cfg, d, dgz, skew_alpha=3.0)
        o2, c2 = gen.gen_csr(cfg.n_nodes, cfg.avg_degree, cfg.seed, skew_alpha=3.0)
        ok_csr = bool(e == o2[-1] and np.array_equal(off, o2) and np.array_equal(col, c2))
        counts = np.bincount(col, minlength=cfg.n_nodes)
        skewed = bool(np.sort(counts)[::-1][: cfg.n_nodes // 100].sum() > 0.1 * col.shape[0])
        d.barrier()
        for x in bufs:
            x.free()
        d.close()
        q.put((rank, "dev_shm_free_gb" in ok_small if rank == 0 else True, raised, ok_csr, skewed))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), None, False, False))


def test_preflight_and_skewed_csr_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_preflight_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for rank, ok_small, raised, ok_csr, skewed in res:
        assert ok_small is True, ok_small
        assert raised and "host RAM" in raised, (rank, raised)
        assert ok_csr and skewed


def test_cpu_helpers():
    assert bench._parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    allowed = sorted(os.sched_getaffinity(0))
    assert bench.node_cpus(-1) == allowed
    assert set(bench.node_cpus(0)) <= set(allowed)
    before = os.sched_getaffinity(0)
    with bench.pinned_threads(allowed[:1]):
        assert os.sched_getaffinity(0) == {allowed[0]}
    assert os.sched_getaffinity(0) == before


def _args(**kw):
    a = dict(config=4, row_bytes=512, base=0, dtype="f32", cache_frac=0.0, skew_alpha=3.0)
    a.update(kw)
    return argparse.Namespace(**a)


def test_workload_label_is_the_same_in_both_arms():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["config"]["workload"] == bench.workload_name(_args(config=1))
    assert "config5" in bench.workload_name(_args(config=5, row_bytes=66, dtype="f16", base=4))
    assert "cached" in bench.workload_name(_args(cache_frac=0.2))


def test_chrome_trace(tmp_path):
    tl = {"shape": {"fetch_sms": 32}, "steps": [{"step": 0, "sample": [0.0, 0.3], "gather": [0.3, 9.0],
                                                 "consume": [0.1, 8.0]}]}
    p = tmp_path / "t.json"
    bench.write_chrome_trace(str(p), tl)
    d = json.loads(p.read_text())
    xs = [e for e in d["traceEvents"] if e["ph"] == "X"]
    assert len(xs) == 3 and {e["tid"] for e in xs} == {1, 2, 3}
    g = [e for e in xs if e["name"] == "gather 0"][0]
    assert g["ts"] == 300.0 and abs(g["dur"] - 8700.0) < 1e-6


def test_reference_arm_config5():
    """The reference arm on a config-5 point (fp16 rows of an odd dim at a 4-byte base offset), on a
    shrunken host buffer: the oracle gathers a bounded sample of the same lists our arm times."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "5",
                        "--row-bytes", "66", "--dtype", "f16", "--base", "4", "--table-gb", "0.5", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["cores"] == 1
    assert line["config"]["workload"] == bench.workload_name(_args(config=5, row_bytes=66, dtype="f16", base=4,
                                                                    table_gb=0.5))
