"""Summarise an ncu --page source --print-source sass export of one kernel: instructions per
member pass, issue, stall reasons, and the top stall-sampled instructions.
    python scripts/src_stats.py gpurun_out/x.ncu-rep [passes] [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
passes = float(sys.argv[2]) if len(sys.argv) > 2 else 4e6
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, data = rows[1], rows[2:]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
samp = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ia]) for r in data)
S = sum(int(r[samp]) for r in data)
print(rows[0][1][:110])
print(f"warp instructions {tot:.4g}, per pass {tot / passes:.1f}, stall samples {S}")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
t = {c: sum(int(r[h.index(c)]) for r in data) for c in cols}
print("  ".join(f"{c[6:]} {v / S * 100:.1f}%" for c, v in sorted(t.items(), key=lambda x: -x[1])[:8]))
for k in sorted(range(len(data)), key=lambda k: -int(data[k][samp]))[:top]:
    print(f"{k:5d} {int(data[k][ia]):9d} {int(data[k][samp]):6d}  {data[k][isrc].strip()[:70]}")
