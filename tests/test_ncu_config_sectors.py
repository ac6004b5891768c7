"""The committed ncu captures of one bench gather per config (profiles/r01/ncu_gather_summary.json:
launch 4 of `bench.py --config c --steps 3 --warmup 3`, i.e. global batch j = 3) read exactly the
sectors the oracle's request model predicts for that minibatch: the distinct 32 B sectors of each
32-row batch of the address-sorted U (merged plan), U drawn by the oracle sampler.  CPU only."""
import json
import os

import numpy as np
import pytest

import dgz_inputs as gen
import oracle
from oracle import request_model as rm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cid", [2, 3, 4])
def test_ncu_sysmem_sectors_match_request_model(cid):
    with open(os.path.join(ROOT, "profiles", "r01", "ncu_gather_summary.json")) as f:
        cap = json.load(f)[f"config{cid}"]
    src = cap["source"]     # config 4 is bench.py's default (no --config flag in its command)
    assert (f"--config {cid}" in src or f"(config {cid}," in src) and "--warmup 3" in src and "launch 4" in src
    c = gen.CONFIGS[cid]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    j = 3
    s = oracle.sample_uniform(off, col, gen.batch_seeds(c.n_nodes, c.batch, c.seed, j), c.fanouts,
                              gen.batch_rng_seed(c.seed, j), with_blocks=False)
    srt = np.sort(s.U)
    R = c.row_bytes
    want = rm.merged_plan_sectors(srt.tolist(), R)
    assert cap["sysmem_read_sectors"] == want, (cap["sysmem_read_sectors"], want)
    # and never below the useful bytes: sectors * 32 >= |U| * R
    assert cap["sysmem_read_sectors"] * 32 >= srt.shape[0] * R
