import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models, graph
g = models.resnet(18, hw=60, classes=16, width=64)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=3, dtype="bf16", fuse_epilogue=True, use_graph=False))
print([(s.kind, s.family, s.output) for s in m.steps[:4]], flush=True)
m.set_inputs({"x": np.random.default_rng(0).uniform(-1, 1, (3, 3, 60, 60)).astype(np.float32)})
m.run(); m.sync(); print("ok", flush=True)
