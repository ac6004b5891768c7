"""Summarise an ncu launch list (gpu__time_duration.sum, --csv) by kernel: count, time, share."""
import collections
import csv
import re
import sys


def short(n):
    m = re.search(r"(\w+_kernel)\b", n)
    return m.group(1) if m else n.split("(")[0][:40]


def main(path, start_kernel="seeds_mark_kernel"):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    seq = [(short(r[ki]), float(r[vi].replace(",", "")) / 1e6) for r in data if r[mi] == "gpu__time_duration.sum"]
    first = [i for i, (n, _) in enumerate(seq) if n == start_kernel][0]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in seq[first:]:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"# {path}: launches from the first {start_kernel} on ({len(seq) - first} launches, {tot:.3f} ms); "
          "ncu serialises launches and runs them cold: compare shares, not absolute times")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} launches={c:4d} total_ms={v:9.3f} per_launch_us={v / c * 1e3:9.1f} share={v / tot * 100:6.2f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
