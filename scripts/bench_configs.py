"""Throughput of the other BASELINE configs at full size (device-timed, inputs resident)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models

CFGS = [
    ("C1 small CNN f32 B=32 32x32", lambda: models.small_cnn(), 32, "f32", 32),
    ("C2 ResNet-18 f32/TF32 B=64 224", lambda: models.resnet(18), 64, "f32", 224),
    ("C5 DenseNet-121 bf16 B=128 224", lambda: models.densenet121(), 128, "bf16", 224),
    ("C5 MobileNet-V2 bf16 B=128 224", lambda: models.mobilenet_v2(), 128, "bf16", 224),
]
for name, build, B, dt, hw in CFGS:
    t0 = time.time()
    try:
        g = build()
        m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype=dt, fuse_epilogue=True))
        x = np.random.default_rng(0).uniform(-1, 1, (B, 3, hw, hw)).astype(np.float32)
        m.set_inputs({"x": x})
        for _ in range(3):
            m.run()
        m.sync(); m.event(0)
        for _ in range(10):
            m.run()
        m.event(1); m.sync()
        ms = m.elapsed_ms(0, 1) / 10
        print(f"{name:36s} {ms:8.3f} ms/step {B / ms * 1e3:10.1f} img/s  units {len(m.units)} (compile {time.time() - t0:.1f}s)", flush=True)
    except Exception as e:
        print(f"{name:36s} FAILED: {type(e).__name__}: {e}", flush=True)
