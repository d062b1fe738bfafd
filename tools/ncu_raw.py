"""Print selected raw metrics from an ncu report (dev tool)."""
import csv, subprocess, sys
rep = sys.argv[1]
pats = sys.argv[2:] or ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active", "lts__t_bytes.sum",
                        "lts__throughput.avg.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "sm__throughput.avg.pct", "smsp__inst_executed.sum", "l1tex__throughput.avg.pct",
                        "sm__warps_active.avg.pct", "smsp__issue_active.avg.pct"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, vals = r[0], r[1], r[2:]
for v in vals:
    for i, name in enumerate(h):
        if any(p in name for p in pats) and not name.endswith(("peak_sustained", "per_second", ".max", ".min")):
            print(f"{name:90s} {v[i]:>20s} {units[i]}")
