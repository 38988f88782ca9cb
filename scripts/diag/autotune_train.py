"""ResNet-50 B=128 bf16 training plan with and without autotune (fprop + dgrad tiles)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2003_10688_b200 import frontend, models
B = 128
g = models.resnet(50, hw=224, classes=1000, train=True)
rng = np.random.default_rng(0)
t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1
ins = {"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32), "t": t}
for tune in (False, True):
    t0 = time.time()
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, lr=0.01, autotune=tune,
                                                      tune_budget=3, cache=False))
    m.set_inputs(ins)
    for _ in range(4):
        m.run()
    m.sync()
    best = 1e9
    for rep in range(3):
        m.event(0)
        for _ in range(10):
            m.run()
        m.event(1)
        m.sync()
        best = min(best, m.elapsed_ms(0, 1) / 10)
    print(f"autotune={tune}: {best:.3f} ms/step ({B / best * 1e3:.0f} img/s), setup {time.time() - t0:.1f}s, "
          f"tuned {len([k for k in m.tuned if k != 'none'])}", flush=True)
    if tune:
        for i, e in sorted((k, v) for k, v in m.tuned.items() if k != "none"):
            c = e["candidates"]
            best_t, auto_t = e["micros"], c.get("0", float("nan"))
            if auto_t - best_t > 2.0:
                print(f"  {m.steps[i].output:34s} tile {e['choice']['tile_n']:3d} {best_t:7.1f} us (heuristic {auto_t:7.1f})")
    del m
