"""Diagnostic: outputs of the fused dgrad + Add + ReluBack units vs the unfused plan (keep_all)."""
import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2003_10688_b200 import frontend, graph, models, dfp
from tests.test_gpu_units import _inputs
from tests.gpu_util import from_device
import torch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = models.resnet(50, hw=224, classes=1000, train=True, seed=11) if B > 8 else models.resnet(18, hw=32, classes=16, width=16, train=True, seed=11)
ins = _inputs(graph.infer_shapes(g, B), B, seed=9)
def opts(**kw):
    return frontend.OptimizeOptions(batch=B, dtype="bf16", train=True, lr=0.0, keep_all=True, cache=False, **kw)
a = frontend.optimize(g, opts())
b = frontend.optimize(g, opts(fuse_relu_back=False))
a.train_step(ins); b.train_step(ins)
pa, pb = a._plan(True), b._plan(True)
def get(m, nm):
    raw = m.read_tensor(nm)
    t = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16)
    return from_device(t, m.graph.meta_of(nm)).astype(np.float64)
for u in pa.units:
    ops = [pa.graph.find_node(n).op for n in u.node_ids]
    if u.kind == "dnn" and ops[0] == "Conv2dBackX" and len(ops) == 3:
        x, y = get(pa, u.output), get(pb, u.output)
        d = np.abs(x - y)
        print(u.output, ops, "max|d|", d.max(), "max|y|", np.abs(y).max(), "nz-diff", int((d > 0).sum()), "of", d.size)
        dx = get(pb, u.node_ids[0])
        oth = get(pb, [i for i in pa.graph.find_node(u.node_ids[1]).inputs if i != u.node_ids[0]][0])
        print("   max|dx|", np.abs(dx).max(), "max|other|", np.abs(oth).max(), "max|dx+other|", np.abs(dx + oth).max())
