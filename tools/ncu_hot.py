"""Per-instruction stall breakdown from an ncu report (source page, SASS)."""
import csv
import subprocess
import sys

path = sys.argv[1]
reason = sys.argv[2] if len(sys.argv) > 2 else None
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.005
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
col = hdr.index(reason) if reason else hdr.index("Warp Stall Sampling (All Samples)")
ia, isrc, ie = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
tot = sum(float(r[col] or 0) for r in data) or 1
print(f"{reason or 'all'}: total {tot:.0f}")
for r in data:
    w = float(r[col] or 0)
    if w / tot > thr:
        print(f"{r[ia][-5:]:>6} {100 * w / tot:5.1f}% {r[ie]:>10} {r[isrc][:100]}")
