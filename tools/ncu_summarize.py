"""Summarise ncu captures into profiles/ (run here, after gpurun brought the
.ncu-rep / launch-list CSV back in gpurun_out/).

    python tools/ncu_summarize.py --round r01 --tag v5 \
        --full gpurun_out/full_*.ncu-rep --launches gpurun_out/launches.csv

Writes profiles/<round>/ncu_full_<tag>_summary.csv (one row per captured
kernel: time, DRAM bytes, L2 hit rate, occupancy, issue, top stall reasons),
profiles/<round>/launches_<tag>_summary.csv (mean us and share per kernel of
the launch list) and merges per-launch DRAM traffic into
profiles/traffic.json, which bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__grid_size", "launch__block_size", "sm__inst_executed.sum",
]


def short(name):
    n = name.split("(")[0]
    for pre in ("void ", "unnamed>::", "s2d::", "<unnamed>::"):
        n = n.replace(pre, "")
    return n


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    return [dict(zip(h, r), _units=units) for r in rows[2:]]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def stall_top(rep, k=4):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return ""
    h = rows[1]
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not" not in c]
    tot = defaultdict(int)
    for r in rows[2:]:
        for i in cols:
            try:
                tot[h[i][6:]] += int(r[i])
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1
    return " ".join(f"{n}:{100 * v / s:.0f}%" for n, v in sorted(tot.items(), key=lambda t: -t[1])[:k])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--tag", required=True)
    ap.add_argument("--full", nargs="*", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--exclude", nargs="*", default=["k_init_rows"], help="setup kernels left out of the shares")
    a = ap.parse_args()
    od = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(od, exist_ok=True)
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = {}
    if os.path.exists(traffic_path):
        traffic = json.load(open(traffic_path))
    if a.full:
        with open(os.path.join(od, f"ncu_full_{a.tag}_summary.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel"] + METRICS + ["top_stalls"])
            for rep in a.full:
                st = stall_top(rep)
                for r in raw_rows(rep):
                    name = short(r.get("Kernel Name", "?"))
                    w.writerow([name] + [r.get(m, "") for m in METRICS] + [st])
                    try:
                        u = r["_units"]
                        rd = float(r["dram__bytes_read.sum"]) * SCALE[u["dram__bytes_read.sum"]]
                        wr = float(r["dram__bytes_write.sum"]) * SCALE[u["dram__bytes_write.sum"]]
                        traffic[name.split("<")[0]] = {"dram_bytes_per_launch": rd + wr, "read_bytes": rd,
                                                       "write_bytes": wr, "source": os.path.basename(rep),
                                                       "round": a.round, "tag": a.tag}
                    except (KeyError, ValueError):
                        pass
        json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        unit_i = h.index("Metric Unit") if "Metric Unit" in h else None
        d = defaultdict(list)
        for r in rows[hi + 1:]:
            if len(r) > vi:
                v = float(r[vi].replace(",", ""))
                u = r[unit_i] if unit_i is not None else "ns"
                v = v / 1000.0 if u == "ns" else (v * 1000.0 if u == "ms" else v)
                k = short(r[ki])
                if not any(k.startswith(x) for x in a.exclude):
                    d[k].append(v)
        total = sum(sum(v) for v in d.values()) or 1
        with open(os.path.join(od, f"launches_{a.tag}_summary.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "launches", "mean_us", "total_us", "share_of_listed"])
            for k, v in sorted(d.items(), key=lambda t: -sum(t[1])):
                w.writerow([k, len(v), f"{sum(v) / len(v):.1f}", f"{sum(v):.1f}", f"{sum(v) / total:.3f}"])


if __name__ == "__main__":
    main()
