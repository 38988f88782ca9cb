#!/usr/bin/env python3
"""Summarise ncu CSV logs into markdown tables for profiles/ (launch list share per kernel; per
launch DRAM traffic of the conv kernel)."""
import csv
import re
import sys
from collections import OrderedDict


def rows(path):
    with open(path) as f:
        return list(csv.DictReader(l for l in f if l.startswith('"')))


def short(name):
    name = re.sub(r"\(.*$", "", name.replace("void ", "").replace("(anonymous namespace)::", ""))
    return name.replace("unnamed>::", "")[:70]


def by_launch(path):
    out = OrderedDict()
    for r in rows(path):
        d = out.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return out


def launch_table(path):
    L = by_launch(path)
    agg = OrderedDict()
    for d in L.values():
        a = agg.setdefault(short(d["name"]), [0, 0.0])
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"]
    tot = sum(a[1] for a in agg.values())
    print(f"{len(L)} launches, {tot/1e6:.3f} ms total (serialised, cold-cache under ncu)\n")
    print("| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t/1e6:.3f} | {100*t/tot:.1f}% |")


def traffic_table(path):
    L = by_launch(path)
    print("| # | kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s |\n|---:|---|---:|---:|---:|---:|")
    for i, d in L.items():
        t = d["gpu__time_duration.sum"]
        rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
        print(f"| {i} | `{short(d['name'])}` | {t/1e3:.1f} | {rd/1e6:.1f} | {wr/1e6:.1f} | {(rd+wr)/t:.0f} |")


def traffic_json(path, out):
    """Mean DRAM bytes per launch of the conv kernels in an ncu metrics CSV (for bench.py)."""
    import json
    L = by_launch(path)
    vals = [d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in L.values()]
    with open(out, "w") as f:
        json.dump({"source": path, "launches": len(vals), "mean_dram_bytes_per_launch": sum(vals) / max(1, len(vals)),
                   "note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per conv launch, one inference step"}, f)


def family_traffic_table(path, peak_gbs=6551.4):
    """Per-kernel totals of an ncu time + DRAM metrics CSV: DRAM GB/s against the measured HBM
    copy peak (MEASURED_PEAKS.json); cold-cache, serialised launches."""
    L = by_launch(path)
    agg = OrderedDict()
    for d in L.values():
        a = agg.setdefault(short(d["name"]), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["gpu__time_duration.sum"]
        a[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    tot = sum(a[1] for a in agg.values())
    print(f"{len(L)} launches, {tot/1e6:.3f} ms total (serialised, cold-cache under ncu)\n")
    print("| kernel | launches | total ms | DRAM MB | DRAM GB/s | of HBM peak |\n|---|---:|---:|---:|---:|---:|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t/1e6:.3f} | {b/1e6:.0f} | {b/t:.0f} | {100*b/t/peak_gbs:.0f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "traffic-json":
        traffic_json(sys.argv[2], sys.argv[3])
    else:
        {"launches": launch_table, "traffic": traffic_table, "family-traffic": family_traffic_table}[sys.argv[1]](sys.argv[2])
