"""Compare every unit output of a compiled plan with the oracle (all buffers kept)."""
import sys
sys.path.insert(0, '.')
import numpy as np
from oracle import sol_oracle as O
from paper_2003_10688_b200 import frontend, graph, autodiff, dfp
from tests.test_gpu_units import _graphs, _inputs
from tests.gpu_util import from_device
name = sys.argv[1] if len(sys.argv) > 1 else "resnet18"
dtype = sys.argv[2] if len(sys.argv) > 2 else "bf16"
batch = 8
g = _graphs()[name](True)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype=dtype, train=True, lr=0.0, keep_all=True))
ins = _inputs(graph.infer_shapes(g, batch), batch, seed=9)
m.train_step(ins)
env = O.run_graph(m.graph, ins)
import torch
for u in m.units:
    meta = m.graph.meta_of(u.output)
    raw = m.read_tensor(u.output)
    f32 = dfp.is_f32_tensor(m.graph, u.output) or dtype == "f32"
    t = torch.from_numpy(raw.view(np.float32) if f32 else raw.view(np.int16).copy()).view(torch.float32 if f32 else torch.bfloat16)
    got = from_device(t, meta)
    err = O.oracle_err(got, env[u.output])
    flag = "  <<<<" if err > 0.05 else ""
    print(f"{u.output:40s} {'/'.join(m.graph.find_node(i).op for i in u.node_ids):40s} {err:.3e}{flag}")
