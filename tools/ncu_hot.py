"""Top SASS lines by warp-stall samples from an ncu report (source page, --print-source sass).
    python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ci = {k: i for i, k in enumerate(hdr)}
k = "Warp Stall Sampling (All Samples)"
data = []
for r in rows[2:]:
    try:
        data.append((float(r[ci[k]]), r[ci["Address"]][-5:], r[ci["Source"]].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d for d, _, _ in data) or 1
for d, a, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * d / tot:5.1f}%  {a}  {s}")
