"""Top SASS lines by warp-stall samples from an ncu report (run here, no GPU)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
i = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    try:
        data.append((float(r[i]), r[0][-5:], r[1].strip()[:100]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for v, a, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * v / tot:5.1f}%  {a}  {s}")
