"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
per-kernel launch count, total time and share of the step (dev tool).
usage: launch_summary.py launches.csv [header line]"""
import csv, sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
    name = r[ix["Kernel Name"]][:60]
    tot[name] += ms
    cnt[name] += 1
all_ms = sum(tot.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{name:60s} launches={cnt[name]:3d} total_ms={ms:10.3f} share={100 * ms / all_ms:5.1f}%")
