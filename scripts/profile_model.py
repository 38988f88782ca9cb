"""Per-family / top-step device times of one model's inference plan: profile_model.py <name> [B]."""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models
name = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
g = {"densenet": lambda: models.densenet121(), "mobilenet": lambda: models.mobilenet_v2(),
     "resnet18": lambda: models.resnet(18), "resnet50": lambda: models.resnet(50)}[name]()
dt = sys.argv[3] if len(sys.argv) > 3 else "bf16"
m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype=dt, fuse_epilogue=True))
m.set_inputs({"x": np.random.default_rng(0).uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)})
m.run(); m.run(); m.sync()
times = m.profile(); times = m.profile()
tot = sum(times)
print(f"total {tot/1e3:.3f} ms over {len(times)} steps")
fam = {}
for st, t in zip(m.steps, times):
    a = fam.setdefault(st.family, [0, 0]); a[0] += t; a[1] += 1
for f, (t, n) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
    print(f"{f:28s} {t/1e3:8.3f} ms {n:4d} steps {100*t/tot:5.1f}%")
rows = sorted(zip(times, m.steps), key=lambda r: -r[0])[:15]
for t, st in rows:
    ops = "+".join(m.graph.find_node(n).op for n in st.node_ids) if st.node_ids else ""
    print(f"{t:8.1f} us {st.family:26s} {st.output:28s} {ops[:50]:50s} {st.algo_bytes / max(t, 1e-9) / 1e3:7.0f} GB/s")
