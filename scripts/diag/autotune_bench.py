"""ResNet-50 B=256 bf16 inference plan with and without autotune: step time and the chosen tiles."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2003_10688_b200 import frontend, models

g = models.resnet(50, hw=224, classes=1000)
x = np.random.default_rng(0).uniform(-1, 1, (256, 3, 224, 224)).astype(np.float32)
for tune in (False, True):
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=256, dtype="bf16", fuse_epilogue=True, autotune=tune,
                                                      tune_budget=5, cache=False))
    m.set_inputs({"x": x})
    for _ in range(5):
        m.run()
    m.sync()
    best = 1e9
    for rep in range(3):
        m.event(0)
        for _ in range(20):
            m.run()
        m.event(1)
        m.sync()
        best = min(best, m.elapsed_ms(0, 1) / 20)
    print(f"autotune={tune}: {best:.3f} ms/step  {256 / best * 1e3:.0f} img/s", flush=True)
    if tune:
        for i, e in sorted(m.tuned.items()):
            if i == "none":
                continue
            st = m.steps[i]
            c = e["candidates"]
            print(f"  {st.output:14s} tile {e['choice']['tile_n']:3d}  " + "  ".join(f"{k}:{v:.1f}" for k, v in c.items()))
    del m
