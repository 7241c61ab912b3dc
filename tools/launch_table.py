"""Per-launch table of an `ncu --metrics gpu__time_duration.sum --csv` log:
kernel, grid, microseconds (the last `--last` launches)."""
import csv
import io
import sys


def rows(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    return [r for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))) if r["Metric Name"] == "gpu__time_duration.sum"]


if __name__ == "__main__":
    rs = rows(sys.argv[1])
    last = int(sys.argv[2]) if len(sys.argv) > 2 else len(rs)
    tot = 0.0
    for r in rs[-last:]:
        name = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("void ", "")
        us = float(r["Metric Value"]) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        tot += us
        print(f"{name[:70]:70s} {r['Grid Size']:>14s} {us:9.1f}")
    print(f"{'total':70s} {'':>14s} {tot:9.1f}")
