"""Aggregate ncu warp-stall samples per CUDA source line (dev tool).
usage: ncu_lines.py report.ncu-rep [top]"""
import csv, collections, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cnt, src, reasons = collections.Counter(), {}, collections.defaultdict(collections.Counter)
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if not hdr or len(r) < 6 or not r[0]:
        continue
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    cnt[key] += s
    src.setdefault(key, r[1].strip()[:70])
    for h, i in hdr.items():
        if h.startswith("stall_") and i < len(r) and r[i]:
            try:
                reasons[key][h[6:]] += int(r[i])
            except ValueError:
                pass
tot = sum(cnt.values())
print("total samples", tot)
for k, v in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{v:8d} {100*v/tot:5.1f}% {k[0]}:{k[1]:<5d} {src[k]:70s} {reasons[k].most_common(2)}")
