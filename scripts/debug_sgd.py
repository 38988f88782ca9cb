import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import sol_oracle as O
from paper_2003_10688_b200 import frontend, graph, models, autodiff
from tests.test_gpu_units import _inputs
batch=16; lr=float(sys.argv[1]) if len(sys.argv)>1 else 0.05
g = models.small_cnn(train=True, hw=32)
gi = graph.infer_shapes(g, batch); ins = _inputs(gi, batch, seed=9)
tg = autodiff.build_training_graph(gi); tgi = graph.infer_shapes(tg.graph, batch)
# oracle SGD trajectory
p = {k: v.astype(np.float64) for k, v in g.params.items()}
ol = []
for it in range(4):
    gg = tgi.copy(); gg.params = {k: v.astype(np.float32) for k, v in p.items()}
    env = O.run_graph(gg, ins); ol.append(float(env[tg.loss]))
    for pn, gn in tg.param_grads: p[pn] = p[pn] - lr * env[gn]
m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=True, lr=lr))
ml = [m.train_step(ins) for _ in range(4)]
print("oracle", ol); print("b200  ", ml)
mf = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=True, lr=lr, use_graph=False))
print("b200 eager", [mf.train_step(ins) for _ in range(4)])
