"""Per-step times of the ResNet-50 B=256 fused inference plan's GEMM steps with parts of the
conv kernels switched off: run once per SOL_CONV_DBG value (1 no output stores, 2 no MMAs,
3 neither), e.g. for d in 0 1 2 3; do SOL_CONV_DBG=$d python scripts/diag/dual_modes.py; done"""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models
B = 256
g = models.resnet(50, hw=224, classes=1000)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", fuse_epilogue=True))
rng = np.random.default_rng(0)
m.set_inputs({"x": rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)})
m.run(); m.sync()
want = sys.argv[1:] or ["l1.0.relu", "l2.0.relu", "l3.0.relu", "l4.0.relu", "l1.1.relu", "l2.1.relu", "l3.1.relu",
                        "l2.1.relu1", "l3.1.relu1", "l2.0.relu1", "l3.0.relu2", "l4.1.relu2"]
m.profile()
times = dict(zip([st.output for st in m.steps], m.profile()))
print(f"SOL_CONV_DBG={os.environ.get('SOL_CONV_DBG', '0')}: " + " ".join(f"{o}={times[o]:.1f}" for o in want if o in times))
