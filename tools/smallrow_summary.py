"""Summarise the small-row study (profiles/r02/smallrow_study.jsonl + the ncu capture of the same
launches, profiles/r02/smallrow_ncu.csv) into profiles/r02/smallrow_walks.json: per point the rows/s,
the distinct 64 KiB regions/s, and the page-walk traffic (L2 sectors no SM issued = all L2 sectors
minus those from the GPCs, the other die's L2 fabric and the GCC; DRAM reads) per distinct region.

    python tools/smallrow_summary.py
"""
import csv
import json
import os

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(HERE, "profiles", "r02")


def ncu_launches(path):
    hdr, out = None, {}
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.setdefault(int(d["ID"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return [out[k] for k in sorted(out)]


def main():
    timing = [json.loads(l) for l in open(os.path.join(P, "smallrow_study.jsonl"))]
    launches = ncu_launches(os.path.join(P, "smallrow_ncu.csv"))
    # the ncu run (--ncu) made one launch per point in the same order: part A strides, then part B widths.
    # Its part-A lists can be shorter (the table cursor advances differently), so rows come from the
    # launch's own sysmem sectors; part-B lists are the timing run's (same seeds)
    assert len(launches) == len(timing)
    pts = []
    for t, m in zip(timing, launches):
        rows = m["syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum"] / (t["R"] // 32)
        other = (m["lts__t_sectors.sum"] - m["lts__t_sectors_srcnode_gpc.sum"] - m["lts__t_sectors_srcunit_ltcfabric.sum"]
                 - m["lts__t_sectors_srcunit_gcc.sum"])
        if t["part"] == "A":   # fixed stride s: one 64 KiB region per 65536 / s rows (one per row from 64 KiB up)
            regions = rows * min(1.0, t["stride"] / 65536.0)
        else:
            regions = t["regions64k"]
        pts.append({"part": t["part"], "R": t["R"], "stride": t.get("stride"), "mrows_s": t["mrows_s"], "gbs": t["gbs"],
                    "m_regions64k_s": t["m_regions64k_s"], "ncu_rows": int(round(rows)), "ncu_regions64k": int(round(regions)),
                    "walk_l2_sectors_per_region": round(other / max(regions, 1), 2),
                    "dram_read_bytes_per_region": round(m["dram__bytes_read.sum"] / max(regions, 1), 1),
                    "ncu_ms": round(m["gpu__time_duration.sum"] / 1e6, 3)})
    b = [p for p in pts if p["part"] == "B" and p["R"] <= 512]
    rates = [p["m_regions64k_s"] for p in b]
    mean = sum(rates) / len(rates)
    out = {"points": pts,
           "walker_bound": {"m_regions64k_s_random_R64_512": rates, "mean": round(mean, 1),
                            "spread": round((max(rates) - min(rates)) / mean, 3),
                            "walk_l2_sectors_per_region_random": [p["walk_l2_sectors_per_region"] for p in b],
                            "dram_read_bytes_per_region_random": [p["dram_read_bytes_per_region"] for p in b],
                            "what": "distinct 64 KiB regions of the table translated per second: one GPU page walk per "
                                    "region (a 128 B line of 16 x 8 B PTEs of 4 KiB pages); constant across row widths "
                                    "64-512 B, so rows/s = this rate x rows per distinct 64 KiB region"},
           "how": "tools/smallrow_study.py (timing, CUDA events) and the same script under ncu --metrics (one launch per "
                  "point); walk traffic = lts__t_sectors - srcnode_gpc - srcunit_ltcfabric - srcunit_gcc"}
    with open(os.path.join(P, "smallrow_walks.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out["walker_bound"]))
    for p in pts:
        print(p)


if __name__ == "__main__":
    main()
