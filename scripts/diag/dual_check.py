"""Diagnostic: fused dual-GEMM bottleneck tail vs the unfused plan's block output (keep_all)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2003_10688_b200 import frontend, graph
from paper_2003_10688_b200.models import _bottleneck, _head
from tests.gpu_util import from_device
from tests.test_gpu_units import _inputs
from oracle import sol_oracle as O


def get(m, nm):
    raw = m.read_tensor(nm)
    t = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16)
    return from_device(t, m.graph.meta_of(nm)).astype(np.float64)


def run(cin, width, hw, stride, batch):
    b = graph.GraphBuilder(41)
    b.input("x", graph.meta_nchw(0, cin, hw, hw))
    y, cout = _bottleneck(b, "x", cin, width, stride, "blk")
    y = b.conv("tail", y, cout, 64, 1, 1, 0)
    p = b.gap("gap", y)
    g = _head(b, p, 64, 10, False)
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=17)
    fused = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True, keep_all=True))
    plain = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True, keep_all=True))
    fused.predict(ins)
    u = next(x for x in fused.units if len(x.node_ids) >= 5)
    a = get(fused, u.output)
    env = O.run_graph(gi, ins)
    want = env[u.output]
    err = O.oracle_err(a, want)
    d = np.abs(a - want)
    bad = d > 0.05 * np.abs(want).max()
    idx = np.argwhere(bad)
    print(f"cin={cin} width={width} hw={hw} s={stride} B={batch} out={u.output} err={err:.3e} bad={bad.sum()}/{bad.size}",
          "channels", np.unique(idx[:, 1])[:20] if len(idx) else "", "pixels n", np.unique(idx[:, 0])[:10] if len(idx) else "",
          "rows", np.unique(idx[:, 2])[:20] if len(idx) else "", flush=True)


for env in ("1", "0"):
    os.environ["SOL_DUAL_BN256"] = env
    print("SOL_DUAL_BN256", env)
    for cfg in [(512, 256, 28, 2, 8), (1024, 512, 14, 2, 8), (256, 128, 56, 2, 4), (64, 64, 16, 1, 4), (512, 256, 28, 2, 64),
                (1024, 512, 14, 2, 64)]:
        run(*cfg)
