"""Summarise ncu captures into text files under profiles/ (committed evidence).

    python tools/summarize_ncu.py <round-tag> <launches.csv> <rep1.ncu-rep> [...]

* launches.csv (from `ncu --metrics gpu__time_duration.sum --csv`): per-kernel
  launch count, total/avg device time and share of the step (cold-cache and
  serialised, so compare SHARES, not absolutes).
* each .ncu-rep (from `ncu --set full`): the details page plus the DRAM byte
  counters that define roofline.traffic.
"""
import csv
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles")


def short(name: str) -> str:
    m = re.search(r"::(\w+?)(<[^>]*>)?\(", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def launches(tag, path):
    agg = defaultdict(lambda: [0, 0.0])
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, im, iv, iu = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Value"), hdr.index("Metric Unit"))
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        if r[iu] == "usecond":
            v *= 1e3
        elif r[iu] == "msecond":
            v *= 1e6
        a = agg[short(r[ik])]
        a[0] += 1
        a[1] += v
    total = sum(a[1] for a in agg.values())
    out = os.path.join(OUT, f"{tag}_launches.txt")
    with open(out, "w") as fh:
        fh.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, {path}\n")
        fh.write("# cold-cache, serialised launches: compare shares, not absolute times\n")
        fh.write(f"{'kernel':58s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}\n")
        for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{k:58s} {c:8d} {ns/1e3:10.1f} {ns/1e3/c:9.2f} {100*ns/total:6.1f}%\n")
        fh.write(f"{'TOTAL':58s} {sum(a[0] for a in agg.values()):8d} {total/1e3:10.1f}\n")
    print("wrote", out)


def rep(tag, path):
    base = os.path.splitext(os.path.basename(path))[0]
    det = subprocess.run(["ncu", "-i", path, "--page", "details"], capture_output=True,
                         text=True).stdout
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    keep = {}
    if len(rows) > 2:
        hdr, units, vals = rows[0], rows[1], rows[2]
        for i, h in enumerate(hdr):
            if (h.startswith("dram__bytes_read.sum") or h.startswith("dram__bytes_write.sum")
                    or h in ("gpu__time_duration.sum", "launch__registers_per_thread",
                             "launch__grid_size", "launch__block_size",
                             "sm__warps_active.avg.pct_of_peak_sustained_active",
                             "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
                    or (h.startswith("smsp__average_warps_issue_stalled")
                        and h.endswith("per_issue_active.ratio"))):
                keep[h] = (vals[i], units[i])
    out = os.path.join(OUT, f"{tag}_{base}.txt")
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on: {path}\n\n")
        fh.write("## selected raw metrics\n")
        for k, (v, u) in keep.items():
            fh.write(f"{k} = {v} {u}\n")
        fh.write("\n## details page\n")
        fh.write(det)
    print("wrote", out)


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(OUT, exist_ok=True)
    for p in sys.argv[2:]:
        if p.endswith(".csv"):
            launches(tag, p)
        else:
            rep(tag, p)
