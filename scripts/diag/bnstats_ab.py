"""Per-step times of the ResNet-50 B=128 training plan with (default) and without
(SOL_NO_BN_STATS_EPI=1) BN statistics from the conv epilogue: the forward conv and its BN unit
side by side. Run twice (once per setting) and pass the two outputs to --compare."""
import json
import os
import sys
sys.path.insert(0, '.')
import numpy as np
if sys.argv[1:2] == ["--compare"]:
    a, b = (json.load(open(p)) for p in sys.argv[2:4])
    keys = [k for k in a if k in b]
    rows = sorted(((b[k] - a[k], k, a[k], b[k]) for k in keys), reverse=True)
    tot = sum(r[0] for r in rows)
    print(f"total gain {tot:.1f} us (positive = linked faster)")
    for d, k, x, y in rows[:12] + rows[-12:]:
        print(f"{d:8.1f} us  {k:40s} linked {x:7.1f}  pass {y:7.1f}")
    sys.exit(0)
from paper_2003_10688_b200 import frontend, models
B = 128
g = models.resnet(50, hw=224, classes=1000, train=True)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, cache=False))
rng = np.random.default_rng(0)
ins = {"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)}
t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1; ins["t"] = t
p = m._plan(True)
p.set_inputs(ins); p.run(); p.run(); p.sync()
p.profile()
times = p.profile()
out = {st.output: tm for st, tm in zip(p.steps, times) if st.kind == "unit"}
json.dump(out, open(sys.argv[1], "w"))
print("links", p.bn_stats_links, "total", round(sum(times) / 1e3, 3), "ms")
