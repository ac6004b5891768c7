"""The small-row zero-copy gather is bound by GPU page walks, one per distinct 64 KiB region of the
table, checked on the committed B200 records (profiles/r02/smallrow_study.jsonl,
smallrow_ncu.csv; tools/smallrow_study.py, tools/smallrow_summary.py):

- random sorted lists of 64-512 B rows: distinct 64 KiB regions translated per second is the same
  (within 20 %) at every width, while rows/s differ 3x and GB/s 2.4x;
- fixed-stride lists of 128 B rows: 4 KiB pages are not the unit (8 KiB strides run at 325 M pages/s),
  the rate falls to the same ~64 M/s once every row is in its own 64 KiB region;
- ncu: the traffic no SM issued (page walks) is 3.5-7 L2 sectors and ~150-210 B of DRAM reads per
  distinct 64 KiB region -- one 128 B line of 16 PTEs plus upper levels, i.e. every region is walked
  once (the sorted order leaves nothing to merge);
- so rows/s = walk rate x rows per distinct region: the prediction for 128 B rows matches.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import smallrow_summary  # noqa: E402

P = os.path.join(ROOT, "profiles", "r02")


def _points():
    timing = [json.loads(l) for l in open(os.path.join(P, "smallrow_study.jsonl"))]
    return timing, smallrow_summary.ncu_launches(os.path.join(P, "smallrow_ncu.csv"))


def test_walk_rate_is_constant_across_widths():
    timing, _ = _points()
    b = {t["R"]: t for t in timing if t["part"] == "B"}
    rates = [b[R]["m_regions64k_s"] for R in (64, 128, 256, 512)]
    mean = sum(rates) / len(rates)
    assert (max(rates) - min(rates)) / mean < 0.2, rates
    assert b[64]["mrows_s"] > 3 * b[512]["mrows_s"] and b[512]["gbs"] > 2.4 * b[64]["gbs"]
    # rows/s predicted from the walk rate and the list's density (rows per distinct 64 KiB region)
    pred = mean * b[128]["n"] / b[128]["regions64k"]
    assert abs(pred - b[128]["mrows_s"]) / b[128]["mrows_s"] < 0.1, (pred, b[128]["mrows_s"])


def test_unit_is_64k_not_4k():
    timing, _ = _points()
    a = {t["stride"]: t for t in timing if t["part"] == "A"}
    assert a[128]["gbs"] > 45                                  # contiguous rows: the link
    assert a[8192]["m_pages4k_s"] > 250                        # 4 KiB pages at > 250 M/s: not the limit
    far = [a[s]["m_regions64k_s"] for s in (65536, 131072, 1 << 20)]
    assert all(50 < r < 80 for r in far), far                  # one row per region: the walk rate
    assert a[16384]["m_regions64k_s"] > 50 and a[16384]["mrows_s"] > 3 * a[65536]["mrows_s"]


def test_walk_traffic_per_region():
    timing, launches = _points()
    for t, m in zip(timing, launches):
        if t["part"] != "B" or t["R"] > 512:
            continue
        other = (m["lts__t_sectors.sum"] - m["lts__t_sectors_srcnode_gpc.sum"] - m["lts__t_sectors_srcunit_ltcfabric.sum"]
                 - m["lts__t_sectors_srcunit_gcc.sum"])
        per = other / t["regions64k"]
        dram = m["dram__bytes_read.sum"] / t["regions64k"]
        assert 3.5 < per < 7.0, (t["R"], per)
        assert 120 < dram < 230, (t["R"], dram)
        # the SMs' own traffic is the payload: sysmem sectors = rows x R / 32
        assert m["syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum"] == t["n"] * t["R"] // 32


def test_walk_model_predicts_the_config4_gather():
    """The config-4 gather from a registered table sits on the same walker bound: a minibatch (the bench's last
    timed batches, recomputed here by the oracle) touches ~0.53 M distinct 64 KiB regions of the
    56.9 GB table; at the walk rate measured on random lists that is the measured gather time."""
    import numpy as np
    import dgz_inputs as gen
    import oracle
    line = json.load(open(os.path.join(P, "bench_config4_registered.json")))   # the cudaHostRegister'd table
    assert line["config"]["host_table"] == "registered"
    c = gen.CONFIGS[4]
    off, col = gen.gen_csr(c.n_nodes, c.avg_degree, c.seed)
    regions = []
    for b in line["parity"]["batches"]:
        j = b["j"]
        s = oracle.sample_uniform(off, col, gen.batch_seeds(c.n_nodes, c.batch, c.seed, j), c.fanouts,
                                  gen.batch_rng_seed(c.seed, j), with_blocks=False)
        assert s.U.shape[0] == b["rows"]
        regions.append(np.unique((s.U * c.row_bytes) >> 16).shape[0])
    timing, _ = _points()
    rate = sum(t["m_regions64k_s"] for t in timing if t["part"] == "B" and t["R"] <= 512) / 4 * 1e6
    t_walk_ms = float(np.mean(regions)) / rate * 1e3
    t_meas = line["roofline"]["gather_ms_mean"]
    assert 0.5e6 < np.mean(regions) < 0.56e6
    assert abs(t_walk_ms - t_meas) / t_meas < 0.08, (t_walk_ms, t_meas)


def test_managed_table_removes_the_walks():
    """The same study on a DGZ_HOST_MANAGED table (profiles/r02/smallrow_study_managed.jsonl,
    smallrow_ncu_managed.csv): the page-walk traffic is gone -- DRAM reads are the IDs and the inverse
    permutation (16 B per row) and nothing else -- and 128 / 256 B random rows run at the link's
    request rate instead of the walk rate (about 2x and 1.7x the registered table)."""
    P2 = os.path.join(ROOT, "profiles", "r02")
    man = [json.loads(l) for l in open(os.path.join(P2, "smallrow_study_managed.jsonl"))]
    reg = [json.loads(l) for l in open(os.path.join(P2, "smallrow_study.jsonl"))]
    mb = {t["R"]: t for t in man if t["part"] == "B"}
    rb = {t["R"]: t for t in reg if t["part"] == "B"}
    assert mb[128]["gbs"] > 40 and mb[128]["gbs"] > 1.8 * rb[128]["gbs"]
    assert mb[256]["gbs"] > 1.5 * rb[256]["gbs"] and mb[512]["gbs"] >= 0.98 * rb[512]["gbs"]
    # 64 KiB regions per second far above the registered table's walk rate
    assert mb[128]["m_regions64k_s"] > 1.8 * rb[128]["m_regions64k_s"]
    launches = smallrow_summary.ncu_launches(os.path.join(P2, "smallrow_ncu_managed.csv"))
    for t, m in zip([t for t in man if t["part"] == "B"], launches):
        assert abs(m["dram__bytes_read.sum"] - 16 * t["n"]) / (16 * t["n"]) < 0.05, (t["R"], m["dram__bytes_read.sum"])
        assert m["syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum"] == t["n"] * t["R"] // 32
    # fixed strides: no collapse at 64 KiB any more (the unit is 2 MiB pages)
    ma = {t["stride"]: t for t in man if t["part"] == "A"}
    ra = {t["stride"]: t for t in reg if t["part"] == "A"}
    assert ma[65536]["mrows_s"] > 3.5 * ra[65536]["mrows_s"] and ma[131072]["mrows_s"] > 3.5 * ra[131072]["mrows_s"]
