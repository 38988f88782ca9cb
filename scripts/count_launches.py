"""Counts the device kernels one steady-state ResNet-50 inference step launches (torch.profiler /
CUPTI sees kernels launched by libsolb200.so, also inside CUDA graphs) and compares with the
plan's own per-step claim (sum of StepInfo.launches_frozen) that bench.py reports as gpu_launches."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2003_10688_b200 import frontend, models

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
train = "train" in sys.argv
if train:
    m = frontend.optimize(models.resnet(50, train=True), frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, lr=0.1))
else:
    m = frontend.optimize(models.resnet(50), frontend.OptimizeOptions(batch=B, dtype="bf16", fuse_epilogue=True))
x = np.random.default_rng(0).uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)
ins = {"x": x}
if train:
    t = np.zeros((B, 1000), np.float32); t[np.arange(B), np.arange(B) % 1000] = 1; ins["t"] = t
m.set_inputs(ins)
for _ in range(3):
    m.run()
m.sync()
steps = 5
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        m.run()
    m.sync()
    torch.cuda.synchronize()
names = [e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = [n for n in names if "Memcpy" not in n and "Memset" not in n]
print("measured kernels per step:", len(kern) / steps)
print("claimed (sum launches_frozen):", sum(s.launches_frozen for s in m.steps),
      "(sum launches):", sum(s.launches for s in m.steps))
from collections import Counter
print(Counter(n.split("<")[0].split("(")[0] for n in kern).most_common(12))
