"""Soak test: repeated ResNet-50 training steps (CUDA graph) to catch intermittent stalls."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models
B = 128
m = frontend.optimize(models.resnet(50, train=True), frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, lr=0.01))
x = np.random.default_rng(0).uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)
t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1
m.set_inputs({"x": x, "t": t})
n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
t0 = time.time()
for i in range(n):
    m.run()
    if i % 50 == 0:
        m.sync()
        print("iter", i, round(time.time() - t0, 1), flush=True)
m.sync()
print("done", n, flush=True)
