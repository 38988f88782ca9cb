"""Time one training BatchNorm2d unit (statistics + apply) on a [N, C, H, W] bf16 tensor."""
import ctypes as C, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2003_10688_b200 import _lib as L, graph, partition
from paper_2003_10688_b200.dfp import create_module, storage_bytes
from paper_2003_10688_b200.graph import Meta

def bench(N, Cc, H, W, reps=20):
    b = graph.GraphBuilder(3)
    b.input("x", graph.meta_nchw(0, Cc, H, W))
    y = b.batchnorm("bn", "x", Cc, True)
    g = graph.infer_shapes(b.done([y]), N)
    (u,) = partition.partition(g)
    mod = create_module(g, u, 1)
    dev = torch.device("cuda:0")
    x = torch.randn(N * H * W * Cc, device=dev).to(torch.bfloat16)
    ps = [torch.from_numpy(np.asarray(g.params[p], np.float32)).to(dev) for p in u.params]
    out = torch.empty(N * H * W * Cc, dtype=torch.bfloat16, device=dev)
    scratch = torch.zeros(mod.scratch_bytes // 4 + 64, dtype=torch.float32, device=dev)
    args = [x] + ps + [out]
    ptrs = (C.c_void_p * len(args))(*[t.data_ptr() for t in args])
    st = torch.cuda.current_stream().cuda_stream
    run = lambda: L.check(L.lib().sol_b200_module_run(mod.handle, ptrs, len(args), C.c_void_p(scratch.data_ptr()), C.c_void_p(st), 0))
    for _ in range(3): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): run()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    mb = 3 * x.numel() * 2 / 1e6
    print(f"  [{N},{Cc},{H},{W}] {us:7.1f} us  ({mb:.0f} MB: stats read + apply read/write -> {mb / us * 1e-3:.2f} TB/s)", flush=True)

for shape in [(128, 2048, 7, 7), (128, 1024, 14, 14), (128, 512, 28, 28), (128, 256, 56, 56), (128, 64, 56, 56)]:
    bench(*shape)
