"""Per-step profile of MobileNet-V2 / DenseNet-121 bf16 inference at B=128 (bench other_configs plans)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2003_10688_b200 import frontend, models
for name in sys.argv[1:] or ["mobilenet_v2"]:
    g = models.MODELS[name]()
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=128, dtype="bf16", fuse_epilogue=True))
    m.set_inputs({"x": np.random.default_rng(0).uniform(-1, 1, (128, 3, 224, 224)).astype(np.float32)})
    m.run(); m.run(); m.sync()
    times = m.profile(); times = m.profile()
    fam = {}
    for st, t in zip(m.steps, times):
        a = fam.setdefault(st.family, [0.0, 0, 0.0])
        a[0] += t; a[1] += 1; a[2] += st.algo_bytes
    print(name, f"total {sum(times)/1e3:.3f} ms, {len(times)} steps")
    for f, (t, n, b) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
        print(f"  {f:28s} {t/1e3:7.3f} ms {n:4d} steps {b/(t*1e-6)/1e9:7.0f} GB/s")
    rows = sorted(zip(times, m.steps), key=lambda r: -r[0])[:12]
    for t, st in rows:
        ops = "+".join(m.graph.find_node(n).op for n in st.node_ids) if st.node_ids else ""
        print(f"    {t:8.1f} us {st.family:26s} {st.output:20s} {ops[:50]:50s} {st.algo_bytes/(t*1e-6)/1e9:7.0f} GB/s")
