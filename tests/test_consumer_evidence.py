"""The a7 layer's measurements, checked on the committed B200 records (DESIGN.md sections 4 and 5.1):

- the layer runs on the tensor cores: its SASS holds tcgen05 MMAs (UTCHMMA), the commit (UTCBAR), TMEM
  loads (LDTM), the TMEM allocator (UTCATOMSWS) and TMA tensor stores of y (UTMASTG)
  (profiles/r02/sass_sage_tcgen05.txt);
- it is HBM-bound: on the config-4 last hop it moves >= 0.5 of the measured HBM bandwidth in
  algorithmic bytes, the GEMM is a few percent of its time (tensor pipe < 5 % active), and ncu's DRAM
  bytes stay below the algorithmic bytes (re-read neighbour rows hit L2)
  (consumer_roofline.jsonl, ncu_sage_summary.json);
- the shared-memory carveout is what kept it off the fetch's SMs: a one-warp spin kernel on 64 SMs
  stretched it >= 1.4x with the driver's carveout and <= 1.02x with the maximum
  (overlap_attrib_driver_carveout.jsonl, overlap_attrib_carveout_max.jsonl);
- the bench line with the layer as consumer reports the layer's own roofline and >= 0.85 of the fetch
  hidden by the strict definition (bench_config4_sage_ownstream.json).
"""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "r02")


def _jsonl(name):
    return [json.loads(l) for l in open(os.path.join(P, name)) if l.strip().startswith("{")]


def test_layer_sass_is_tcgen05():
    txt = open(os.path.join(P, "sass_sage_tcgen05.txt")).read()
    for op in ("UTCHMMA", "UTCBAR", "LDTM", "UTCATOMSWS", "LDGSTS", "UTMASTG"):
        assert op in txt, op


def test_layer_is_hbm_bound():
    rows = {r["kernel"]: r for r in _jsonl("consumer_roofline.jsonl")}
    sage = rows["sage_mean_linear ctas_per_sm=0"]
    assert sage["hbm_gbs"] / sage["hbm_peak_gbs"] >= 0.5
    # the layer (mean + GEMM + 2x wider output) is no slower per byte than the mean alone
    assert sage["hbm_gbs"] >= rows["aggregate_mean ctas_per_sm=0"]["hbm_gbs"]
    ncu = json.load(open(os.path.join(P, "ncu_sage_summary.json")))
    assert "sage_mean_linear_kernel" in ncu["kernel"]
    assert ncu["dram_read_bytes"] + ncu["dram_write_bytes"] < ncu["algorithmic_bytes"]
    assert ncu["tensor_pipe_active_pct"] < 5.0
    assert ncu["stall_share"]["long_scoreboard"] == max(ncu["stall_share"].values())


def test_carveout_decides_co_residency():
    drv = [r for r in _jsonl("overlap_attrib_driver_carveout.jsonl") if r.get("carveout") == "driver"
           and "consumer" not in r]
    spin64 = [r for r in drv if r["corunner"] == "spin" and r["sms"] == 64][0]
    assert spin64["stretch"] >= 1.4
    mx = _jsonl("overlap_attrib_carveout_max.jsonl")
    for r in mx:
        if r["corunner"] == "spin":
            assert r["stretch"] <= 1.02, r
    # the consumer without shared memory was never kept off by the spin kernel
    mean = [r for r in _jsonl("overlap_attrib_driver_carveout.jsonl") if r.get("consumer", "").startswith("dgz_aggregate_mean")
            and r["corunner"] == "spin"][0]
    assert mean["stretch"] <= 1.02


def test_bench_line_with_the_layer():
    d = json.loads(open(os.path.join(P, "bench_config4_sage_ownstream.json")).read().splitlines()[-1])
    o = d["overlap"]
    assert o["consumer"].startswith("dgz_sage_mean_linear")
    assert o["consumer_roofline"]["kernel"] == "sage_mean_linear_kernel" and o["consumer_roofline"]["frac"] >= 0.5
    assert o["hidden_frac_best"] >= 0.85
    best = o["best"]
    # hidden = 1 - (T_overlap - T_c) / T_fetch, recomputed from the line's own numbers
    assert abs((1 - (best["t_step_overlapped_ms"] - o["t_consumer_ms"]) / o["t_fetch_ms"]) - o["hidden_frac_best"]) < 0.002
    assert best["shape"][3] == "own stream" and best["shape"][4] == "whole GPU"
