"""The round-2 ncu --set full capture of the headline gather (profiles/r02/ncu_gather_summary.json:
launch 4 of `bench.py --steps 3 --warmup 3`) against the oracle and the walk model.  In that command
the pipeline calibration (pipeline.calibrated_fetcher) fetches the 3 warm-up minibatches j = 0, 1, 2
twice per shape, so gather launch 4 is global batch j = 0 again.  CPU only.

- sysmem sectors read = 16 x |U(j = 0)| exactly (512 B rows on a page-aligned table: S(o) = 16 per
  row, zero over-fetch), U drawn by the oracle sampler;
- DRAM reads = the IDs + inverse permutation (16 B per row) + the page walks of the minibatch's
  distinct 64 KiB regions (~110-210 B each, profiles/r02/smallrow_walks.json)."""
import json
import os

import numpy as np

import dgz_inputs as gen
import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_headline_capture_matches_oracle_and_walk_model():
    with open(os.path.join(ROOT, "profiles", "r02", "ncu_gather_summary.json")) as f:
        cap = json.load(f)["config4"]
    assert "launch 4" in cap["source"] and "--warmup 3" in cap["source"]
    c = gen.CONFIGS[4]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    s = oracle.sample_uniform(off, col, gen.batch_seeds(c.n_nodes, c.batch, c.seed, 0), c.fanouts,
                              gen.batch_rng_seed(c.seed, 0), with_blocks=False)
    n = s.U.shape[0]
    assert cap["sysmem_read_sectors"] == 16 * n
    regions = np.unique((s.U * c.row_bytes) >> 16).shape[0]
    walk_bytes = cap["dram_read_bytes"] - 16 * n
    assert 110 < walk_bytes / regions < 210, walk_bytes / regions
    # and HBM writes = the rows (plus write-allocate noise): n * R within 15 %
    assert abs(cap["dram_write_bytes"] - n * c.row_bytes) / (n * c.row_bytes) < 0.15


def test_managed_capture_has_no_walks():
    """The same launch with the default managed host table (key config4_managed): the same sysmem
    sectors (16 x |U|), and DRAM reads = the IDs and the inverse permutation only (16 B per row),
    i.e. no page-walk traffic."""
    with open(os.path.join(ROOT, "profiles", "r02", "ncu_gather_summary.json")) as f:
        caps = json.load(f)
    cap, reg = caps["config4_managed"], caps["config4"]
    assert "managed" in cap["source"] and "launch 4" in cap["source"]
    assert cap["sysmem_read_sectors"] == reg["sysmem_read_sectors"]          # the same minibatch (j = 0)
    n = cap["sysmem_read_sectors"] // 16
    assert abs(cap["dram_read_bytes"] - 16 * n) / (16 * n) < 0.05
    assert reg["dram_read_bytes"] > 5 * cap["dram_read_bytes"]
