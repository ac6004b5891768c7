"""NEXT-1 evidence ("PCIe bytes avoided"): in the committed ncu capture of a cached gather
(profiles/r01/ncu_cache_gather.json, tools/cache_ncu.py), the kernel read over PCIe exactly the
sectors of the rows that missed the HBM cache -- cached rows cost no PCIe bytes.  CPU only."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cached_gather_reads_only_missed_rows_over_pcie():
    d = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_cache_gather.json")))
    m = d["measured"]
    assert d["missed_rows"] + d["hit_rows"] == d["rows"] and d["hit_rows"] > 0.4 * d["rows"]
    assert d["row_bytes"] % 128 == 0                       # 128 B-aligned rows: exactly R/32 sectors each
    assert m["syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss"] == d["missed_rows"] * d["row_bytes"] // 32
    assert m["pcie__read_bytes"] >= d["missed_rows"] * d["row_bytes"]   # payload plus TLP overhead
    assert "gather_segment_kernel" in d["kernel"] and ", 1, 1, long>" in d["kernel"]   # MERGE + CACHED instance
