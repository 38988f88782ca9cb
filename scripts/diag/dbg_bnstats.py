"""Diagnostic: training plans with and without BN statistics from the conv epilogue (keep_all):
first unit outputs that differ, step by step."""
import sys; sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2003_10688_b200 import frontend, graph, models
from tests.test_gpu_units import _inputs
from tests.gpu_util import from_device
g = models.resnet(50, hw=64, classes=16, width=16, train=True, seed=5)
ins = _inputs(graph.infer_shapes(g, 8), 8, seed=10)
def opts(**kw):
    return frontend.OptimizeOptions(batch=8, dtype="bf16", train=True, lr=0.0, keep_all=True, cache=False, **kw)
a = frontend.optimize(g, opts())
b = frontend.optimize(g, opts(bn_stats_from_conv=False))
pa, pb = a._plan(True), b._plan(True)
print("links", pa.bn_stats_links)
def get(m, nm):
    raw = m.read_tensor(nm)
    meta = m.graph.meta_of(nm)
    if raw.dtype == np.float32 or raw.nbytes == 4 * meta.numel:
        return None
    t = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16)
    return from_device(t, meta).astype(np.float64)
for step in range(2):
    la, lb = a.train_step(ins), b.train_step(ins)
    print("step", step, "loss", la, lb)
    shown = 0
    for u in pa.units:
        if u.kind != "dfp":
            continue
        x, y = get(pa, u.output), get(pb, u.output)
        if x is None or y is None:
            continue
        err = np.abs(x - y).max() / max(np.abs(y).max(), 1e-12)
        if err > 1e-4 and shown < 14:
            ops = "+".join(pa.graph.find_node(n).op for n in u.node_ids)
            print("   ", u.output, ops, "rel", round(float(err), 4), "inputs", u.inputs)
            shown += 1
