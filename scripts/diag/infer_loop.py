"""Soak: the bench's ResNet-50 B=256 inference plan (fused, CUDA graph) replayed for many steps with
a progress line every 50 (scripts/diag/hang_hunt.sh-style stall detection)."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
m = frontend.optimize(models.resnet(50), frontend.OptimizeOptions(batch=256, dtype="bf16", fuse_epilogue=True,
                                                                 cache=False, autotune=True, tune_budget=3))
m.set_inputs({"x": np.random.default_rng(0).uniform(-1, 1, (256, 3, 224, 224)).astype(np.float32)})
t0 = time.time()
for i in range(steps):
    m.run()
    if i % 50 == 0:
        m.sync()
        print(f"step {i} {time.time() - t0:.1f}s", flush=True)
m.sync()
print("done", flush=True)
