"""Summarise an `ncu --set full` capture of the gather into profiles/r01/ncu_gather_summary.json."""
import csv
import io
import json
import subprocess
import sys


def main(rep, out_json, key="config4", note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def g(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")), units[i]

    def b(name):
        v, u = g(name)
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    t = g("gpu__time_duration.sum")[0] * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}[g("gpu__time_duration.sum")[1]]
    sect = g("syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum")[0]
    s = {"kernel": next(v for h, v in zip(hdr, vals) if h == "Kernel Name"),
         "source": note, "duration_ms": round(t * 1e3, 3),
         "dram_read_bytes": int(b("dram__bytes_read.sum")), "dram_write_bytes": int(b("dram__bytes_write.sum")),
         "sysmem_read_sectors": int(sect), "sysmem_read_bytes": int(sect * 32),
         "sysmem_payload_gbs": round(sect * 32 / t / 1e9, 2),
         "pcie_read_gbs_incl_overhead": g("pcie__read_bytes.sum.per_second")[0],
         "pcie_write_gbs_read_requests": g("pcie__write_bytes.sum.per_second")[0],
         "registers_per_thread": g("launch__registers_per_thread")[0], "grid": g("launch__grid_size")[0],
         "block": g("launch__block_size")[0],
         "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active")[0]}
    s["dram_bytes_per_launch"] = s["dram_read_bytes"] + s["dram_write_bytes"]
    try:
        j = json.load(open(out_json))
    except Exception:
        j = {}
    if key in j:
        j[key + "_previous"] = j[key]
    j[key] = s
    json.dump(j, open(out_json, "w"), indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
