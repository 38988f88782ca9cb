"""One eager ResNet-50 B=128 training step (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2003_10688_b200 import frontend, models
B = 128
g = models.resnet(50, hw=224, classes=1000, train=True)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, use_graph=False))
rng = np.random.default_rng(0)
t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1
m.set_inputs({"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32), "t": t})
m.run(); m.sync()
print("ok")
