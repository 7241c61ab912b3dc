"""Hottest SASS lines of an ncu capture (warp-stall samples), for reading
a kernel's bottleneck here:  python tools/ncu_hot.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ix = {c: i for i, c in enumerate(h)}
body = rows[2:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
stall_cols = [c for c in h if c.startswith("stall_") or c.endswith("(All Samples)")]
best = sorted(body, key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))[:top]
for r in best:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{100.0 * s / max(tot, 1):5.1f}%  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")
