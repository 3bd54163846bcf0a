"""Top SASS instructions of an ncu report by warp-stall samples, with their
dominant stall reasons (ncu -i REPORT --page source --print-source sass)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
body = "\n".join(lines[1:])
r = list(csv.reader(io.StringIO(body)))
h = r[0]
rows = r[1:]
iS = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(x[iS] or 0) for x in rows)
print(f"total samples {tot:.0f}, instructions {len(rows)}")
agg = {}
for x in rows:
    for i in stall_cols:
        agg[h[i]] = agg.get(h[i], 0) + float(x[i] or 0)
print("stall totals:", ", ".join(f"{k[6:]} {v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
idx = sorted(range(len(rows)), key=lambda k: -float(rows[k][iS] or 0))[:n]
for k in sorted(idx):
    x = rows[k]
    st = sorted(((float(x[i] or 0), h[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{k:5d} {float(x[iS]) / tot:6.1%} ex={x[iE]:>8} {x[1].strip()[:60]:60s} " + " ".join(f"{b}:{a:.0f}" for a, b in st if a > 0))
