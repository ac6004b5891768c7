"""Hardware evidence for the request plan (SURVEY 8(a) a4', 8(c) "pins"): the per-launch ncu counts
committed in profiles/r01/sector_evidence.json (tools/sector_evidence.py on a B200) against the
oracle's request model on the same regenerated IDs.  CPU only: it reads the committed capture.

- SEGMENT (unsorted): sysmem sectors = sum over rows of S(o), L2 requests = sum of L(o) -- the
  per-row minimum (every line a row touches is requested once, with exactly its sectors) -- exact
  up to the few lines two table-adjacent rows of the random list share, which the hardware may or
  may not merge (bounds: distinct lines/sectors of the whole list <= measured <= per-row sums).
- SEGMENT on an address-sorted list with the shared line merged: between the distinct lines /
  sectors of the whole list and those of each 32-row batch (oracle merged_plan_*).
- NAIVE / SHIFT (Listing 2): never fewer sectors or requests than that minimum, and the
  shift never needs more requests than the naive kernel on a 128 B-aligned table.
"""
import json
import os

import dgz_inputs as gen
from oracle import request_model as rm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EVIDENCE = os.path.join(ROOT, "profiles", "r01", "sector_evidence.json")
SEC = "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss"
REQ = "syslts__t_requests_srcunit_tex_aperture_sysmem_op_read"


def _launches():
    with open(EVIDENCE) as f:
        return json.load(f)["launches"]


def test_evidence_covers_widths_and_variants():
    ls = _launches()
    assert {d["R"] for d in ls} >= {100, 400, 480, 512, 516, 1028, 2408}
    assert {d["base"] for d in ls} == {0, 4}
    assert {d["variant"] for d in ls} == {"segment", "naive", "shift", "segment_sorted_merge"}


def test_segment_plan_matches_hardware_counts():
    for d in _launches():
        ids = [int(x) for x in gen.distinct_ids(d["rows"], d["n"], d["seed"])]
        R, base = d["R"], d["base"]
        lines = sum(rm.row_lines(base + i * R, R) for i in ids)
        sectors = sum(rm.row_sectors(base + i * R, R) for i in ids)
        srt = sorted(ids)
        all_lines = rm.merged_plan_requests(srt, R, base, batch=len(srt))     # distinct over the list
        all_secs = rm.merged_plan_sectors(srt, R, base, batch=len(srt))
        assert lines - all_lines <= 8                                         # few shared lines at all
        if d["variant"] == "segment":
            assert "gather_segment_kernel" in d["kernel"]
            assert all_secs <= d[SEC] <= sectors, d
            assert all_lines <= d[REQ] <= lines, d
        elif d["variant"] == "segment_sorted_merge":
            assert all_secs <= d[SEC] <= rm.merged_plan_sectors(srt, R, base), d
            assert all_lines <= d[REQ] <= rm.merged_plan_requests(srt, R, base), d
        else:
            assert "gather_elem_kernel" in d["kernel"]
            assert d[SEC] >= sectors and d[REQ] >= lines, d


def test_shift_needs_no_more_requests_than_naive_when_aligned():
    by = {(d["R"], d["base"], d["variant"]): d for d in _launches()}
    for (R, base, v), d in by.items():
        if v == "shift" and base == 0:
            assert d[REQ] <= by[(R, base, "naive")][REQ], (R, d[REQ], by[(R, base, "naive")][REQ])
