"""Summarise an `ncu --set full` capture of one dgz_sage_mean_linear launch (the a7 layer) into a JSON
record: duration, DRAM bytes vs the algorithmic bytes, L2 hit rate, occupancy, tensor-pipe use and the
warp-stall breakdown (pc sampling).

    python tools/ncu_sage_summary.py gpurun_out/r02b23/ncu_sage.ncu-rep profiles/r02/ncu_sage_summary.json \
        [alg_bytes] [note]
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, out_json, alg_bytes="708556032", note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def g(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")), units[i]

    def b(name):
        v, u = g(name)
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    d, du = g("gpu__time_duration.sum")
    t = d * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}[du]
    stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
              for h, v in zip(hdr, vals) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6] if v > 0}
    s = {"kernel": next(v for h, v in zip(hdr, vals) if h == "Kernel Name")[:80], "source": note,
         "duration_us": round(t * 1e6, 1),
         "dram_read_bytes": int(b("dram__bytes_read.sum")), "dram_write_bytes": int(b("dram__bytes_write.sum")),
         "algorithmic_bytes": int(alg_bytes),
         "l2_hit_rate_pct": round(g("lts__t_sector_hit_rate.pct")[0], 1),
         "registers_per_thread": g("launch__registers_per_thread")[0], "grid": g("launch__grid_size")[0],
         "block": g("launch__block_size")[0],
         "warps_active_pct": round(g("sm__warps_active.avg.pct_of_peak_sustained_active")[0], 1),
         "stall_share": top}
    s["dram_gbs"] = round((s["dram_read_bytes"] + s["dram_write_bytes"]) / t / 1e9, 1)
    s["algorithmic_gbs"] = round(int(alg_bytes) / t / 1e9, 1)
    for name in ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                 "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active"):
        if name in hdr:
            s["tensor_pipe_active_pct"] = round(g(name)[0], 2)
            break
    json.dump(s, open(out_json, "w"), indent=1)
    print(json.dumps(s))


if __name__ == "__main__":
    main(*sys.argv[1:])
