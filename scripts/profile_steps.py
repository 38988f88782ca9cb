"""Per-step device times of a compiled plan (CUDA events around every step)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models
train = len(sys.argv) > 1 and sys.argv[1] == "train"
B = 128 if train else 256
g = models.resnet(50, hw=224, classes=1000, train=train)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", train=train, fuse_epilogue="fuse" in sys.argv))
rng = np.random.default_rng(0)
ins = {"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)}
if train:
    t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1; ins["t"] = t
m.set_inputs(ins); m.run(); m.run(); m.sync()
times = m.profile(); times = m.profile()
rows = []
for st, t in zip(m.steps, times):
    rows.append((t, st.family, st.output, st.algo_flops / max(t, 1e-9) / 1e6, st.algo_bytes / max(t, 1e-9) / 1e3))
tot = sum(times)
print(f"total {tot/1e3:.3f} ms over {len(times)} steps")
fam = {}
for t, f, o, tf, gb in rows:
    a = fam.setdefault(f, [0, 0]); a[0] += t; a[1] += 1
for f, (t, n) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
    print(f"{f:24s} {t/1e3:8.3f} ms  {n:4d} steps  {100*t/tot:5.1f}%")
fam_filter = [a.split("=", 1)[1] for a in sys.argv if a.startswith("family=")]
if fam_filter:
    ops = {}
    for st in m.steps:
        ops[st.output] = "+".join(m.graph.find_node(n).op for n in st.node_ids) if st.node_ids else ""
    print("--- steps of", fam_filter[0])
    for t, f, o, tf, gb in sorted(rows, reverse=True):
        if f == fam_filter[0]:
            print(f"{t:9.1f} us {o:36s} {ops.get(o, ''):40s} {gb:8.1f} GB/s")
    sys.exit(0)
print("--- steps by lost time vs speed of light (max(FLOP/1416T, bytes/6551G))")
sol = []
for st, t in zip(m.steps, times):
    tmin = max(st.algo_flops / 1416e12, st.algo_bytes / 6551e9) * 1e6
    sol.append((t - tmin, t, tmin, st.family, st.output))
for lost, t, tmin, f, o in sorted(sol, reverse=True)[:25]:
    print(f"{lost:8.1f} us lost  {t:8.1f} us  sol {tmin:7.1f} us ({100 * tmin / max(t, 1e-9):4.0f}%)  {f:26s} {o}")
print("--- top 40 steps")
for t, f, o, tf, gb in sorted(rows, reverse=True)[:40]:
    print(f"{t:9.1f} us {f:22s} {o:36s} {tf:8.1f} TF/s {gb:8.1f} GB/s")
