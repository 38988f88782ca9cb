"""Per-unit check inside a composed plan: re-run the oracle for each unit on the plan's own
input buffers and compare with the plan's output buffer (isolates wiring from precision)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from oracle import sol_oracle as O
from paper_2003_10688_b200 import frontend, graph, dfp, models
from tests.test_gpu_units import _inputs
from tests.gpu_util import from_device
name = sys.argv[1]; batch = 16
if name == "small_cnn": g = models.small_cnn(train=True, hw=32)
else: g = models.resnet(18 if name == "resnet18" else 50, hw=64, classes=16, width=16, train=True)
m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=True, lr=0.0, keep_all=True))
ins = _inputs(graph.infer_shapes(g, batch), batch, seed=9)
m.train_step(ins)
def get(nm):
    if nm in m.params:
        return m.params[nm].astype(np.float64)
    meta = m.graph.meta_of(nm)
    raw = m.read_tensor(nm)
    f32 = dfp.is_f32_tensor(m.graph, nm)
    t = torch.from_numpy(raw.view(np.float32).copy() if f32 else raw.view(np.int16).copy())
    if not f32: t = t.view(torch.bfloat16)
    return from_device(t, meta).astype(np.float64)
params = {k: np.asarray(v, np.float64) for k, v in m.params.items()}
bad = 0
for u in m.units:
    local = {nm: get(nm) for nm in u.inputs}
    for nid in u.node_ids:
        n = m.graph.find_node(nid)
        local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
    want = local[u.output]; got = get(u.output)
    err = O.oracle_err(got, want)
    fin = np.all(np.isfinite(got))
    if err > 2e-2 or not fin:
        bad += 1
        print(f"{u.output:40s} {'/'.join(m.graph.find_node(i).op for i in u.node_ids):40s} err={err:.3e} finite={fin}")
print("bad units:", bad, "of", len(m.units))
