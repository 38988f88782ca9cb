"""Per-kernel summary of an ncu --csv list with gpu__time_duration, dram bytes and tensor-pipe
activity (scripts/ncu_train_conv.sh): launches, total ms, DRAM GB/s, time-weighted tensor active."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
k_i, m_i, v_i, u_i, id_i = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
launch = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    launch[r[id_i]][r[m_i]] = (float(r[v_i].replace(",", "")), r[u_i])
    names[r[id_i]] = r[k_i]
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in launch.items():
    nm = re.sub(r"^void |solb200::|\(.*$", "", names[i]).replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    t = m["gpu__time_duration.sum"][0] * scale[m["gpu__time_duration.sum"][1]]
    b = sum(m[k][0] * scale[m[k][1]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in m)
    tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", (0.0, ""))[0]
    a = agg[nm]
    a[0] += 1; a[1] += t; a[2] += b; a[3] += tp * t
tot = sum(a[1] for a in agg.values())
print(f"{len(launch)} launches, {tot:.3f} ms total (serialised under ncu)\n")
print("| kernel | launches | total ms | DRAM GB/s | tensor pipe active |")
print("|---|---:|---:|---:|---:|")
for nm, (n, t, b, tw) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{nm}` | {n} | {t:.3f} | {b / t:.0f} | {tw / t:.1f}% |")
