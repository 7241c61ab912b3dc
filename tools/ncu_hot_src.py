"""Hottest CUDA source lines (warp-stall samples) of an ncu capture built
with -lineinfo:  python tools/ncu_hot_src.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
res, fname = [], ""
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 5 and r[0].isdigit() and r[2] == "-":  # a source line row (aggregated over its SASS)
        try:
            res.append((int(r[4] or 0), fname, int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot = sum(x[0] for x in res)
for s, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100.0 * s / max(tot, 1):5.1f}%  {f}:{ln:<5} {src[:100]}")
