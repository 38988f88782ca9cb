"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ dram__bytes_read/write.sum]) by
kernel: total time, launches, time per launch, DRAM bytes and GB/s."""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "byte": 1, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    k = collections.defaultdict(dict)
    for d in data:
        k[int(d["ID"])]["name"] = d["Kernel Name"]
        k[int(d["ID"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for _, e in sorted(k.items()):
        n = re.sub(r"\(.*", "", e["name"]).strip().replace("solb200::(anonymous namespace)::", "")
        f = fam[n[:64]]
        f[0] += 1
        f[1] += e.get("gpu__time_duration.sum", 0.0)
        f[2] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in fam.values())
    print(f"{len(k)} launches, {tot / 1000:.3f} ms total (serialised under ncu)")
    print("| kernel | launches | total ms | us / launch | DRAM MB | GB/s |")
    print("|---|---:|---:|---:|---:|---:|")
    for n, (c, t, b) in sorted(fam.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"| `{n}` | {c} | {t / 1000:.3f} | {t / c:.1f} | {b / 1e6:.0f} | {b / (t * 1e-6) / 1e9 if t else 0:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
