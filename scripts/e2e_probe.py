"""Probe copy/compute overlap of the pipelined e2e path (R50 B=256 bf16 inference)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, models, _lib as L
B = 256
m = frontend.optimize(models.resnet(50), frontend.OptimizeOptions(batch=B, dtype="bf16", fuse_epilogue=True))
x = np.random.default_rng(0).uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)
m.set_inputs({"x": x})
for _ in range(3):
    m.run()
m.sync()
lib = L.lib()
K = 10
def timed(fn):
    m.sync(); m.event(2); fn(); m.event(3); m.sync()
    return m.elapsed_ms(2, 3) / K
def only_run():
    for _ in range(K): m.run()
def only_h2d():
    for _ in range(K): L.check(lib.sol_b200_plan_h2d(m.plan, m.in_canon["x"], m.pin_in["x"].ptr, 4 * x.size))
def serial():
    for _ in range(K):
        L.check(lib.sol_b200_plan_h2d(m.plan, m.in_canon["x"], m.pin_in["x"].ptr, 4 * x.size)); m.run()
def staged():
    m.stage_inputs()
    for i in range(K):
        m.run()
        if i + 1 < K: m.stage_inputs()
print("run %.3f ms  h2d %.3f ms  serial %.3f ms  staged %.3f ms" % (timed(only_run), timed(only_h2d), timed(serial), timed(staged)))
t0 = time.perf_counter(); staged(); m.sync(); print("host wall staged %.3f ms/step" % ((time.perf_counter() - t0) * 1e3 / K))
def staged_d2h():
    m.stage_inputs()
    for i in range(K):
        m.run()
        if i + 1 < K: m.stage_inputs()
        L.check(lib.sol_b200_plan_d2h(m.plan, m.pin_out["prob"].ptr, m.out_canon["prob"], 4 * 256 * 1000))
print("staged+d2h %.3f ms" % timed(staged_d2h))
def staged_d2h_b():
    m.stage_inputs()
    for i in range(K):
        m.run()
        L.check(lib.sol_b200_plan_d2h(m.plan, m.pin_out["prob"].ptr, m.out_canon["prob"], 4 * 256 * 1000))
        if i + 1 < K: m.stage_inputs()
print("staged+d2h (d2h first) %.3f ms" % timed(staged_d2h_b))
