import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import sol_oracle as O
from paper_2003_10688_b200 import frontend, graph, dfp
from tests.test_gpu_units import _graphs, _inputs
from tests.gpu_util import from_device
batch = 8
for train in (False, True):
    g = _graphs()["resnet18"](train)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=train, lr=0.0, keep_all=True))
    ins = _inputs(graph.infer_shapes(g, batch), batch, seed=9)
    if train: m.train_step(ins)
    else: m.predict(ins)
    env = O.run_graph(m.graph, ins)
    for name in ["x", "stem"]:
        meta = m.graph.meta_of(name)
        raw = m.read_tensor(name)
        t = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16)
        got = from_device(t, meta)
        print(train, name, meta, O.oracle_err(got, env[name]), got.ravel()[:4], env[name].ravel()[:4])
