"""Per-source-line stall breakdown of an ncu report (source page, -lineinfo)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


cur, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    st = {hdr[i][6:]: f(r[i]) for i in range(len(hdr)) if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
    s = f(r[4])
    if s == 0:
        continue
    agg[(cur, ln)] = (s, f(r[7]), r[1].strip()[:70], st)
tot = sum(v[0] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = sorted(v[3].items(), key=lambda kv: -kv[1])[:3]
    rs = " ".join(f"{n}={100 * x / v[0]:.0f}%" for n, x in reasons if x > 0)
    print(f"{k[0][:16]:16s} {k[1]:4d} {100 * v[0] / tot:5.1f}%  [{rs}]  {v[2]}")
