"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launch count,
summed device time and share (cold-cache, serialised under ncu: compare SHARES, not absolutes).

    python tools/ncu_launch_summary.py gpurun_out/launches.csv > profiles/launches_summary.txt
"""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
hdr = rows[hdr_i]
ki, ui, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ki]).strip()
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6, "second": 1e3}.get(unit, 1.0)
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"source: {path}; {sum(cnt.values())} launches, {all_ms:.1f} ms summed device time (ncu, serialised, cold cache)")
print(f"{'kernel':40s} {'launches':>9s} {'total_ms':>11s} {'share':>7s} {'avg_us':>10s}")
for name, ms in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{name[:40]:40s} {cnt[name]:9d} {ms:11.2f} {ms / all_ms:7.3f} {1e3 * ms / cnt[name]:10.1f}")
