"""1x1-conv GEMMs of ResNet-50 (B=256) through sol_b200_conv_fprop: time per launch (and the
error against a torch fp32 GEMM)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
out = []
for (N, Cin, H, W, Cout) in [(256, 128, 28, 28, 512), (256, 256, 14, 14, 1024), (256, 512, 7, 7, 2048),
                             (256, 256, 56, 56, 128), (256, 512, 28, 28, 256)]:
    d = L.ConvDesc(N, Cin, H, W, Cout, H, W, 1, 1, 1, 1, 0, 0, Cin, 1)
    x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
    w = torch.randn(Cout, Cin, 1, 1, device=dev) * 0.05
    b = torch.randn(Cout, device=dev)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
    y = torch.zeros(N, H, W, Cout, dtype=torch.bfloat16, device=dev)
    for _ in range(3):
        L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), b.data_ptr(), y.data_ptr(), 1, st))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(20):
        L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), b.data_ptr(), y.data_ptr(), 1, st))
    ev1.record()
    torch.cuda.synchronize()
    us = ev0.elapsed_time(ev1) / 20 * 1e3
    ref = x.float().reshape(-1, Cin) @ w.reshape(Cout, Cin).float().t() + b
    err = ((y.float().reshape(-1, Cout) - ref).abs().max() / ref.abs().max()).item()
    tf = 2.0 * N * H * W * Cin * Cout / us / 1e6
    out.append(f"M={N*H*W} K={Cin} N={Cout}: {us:.1f} us {tf:.0f} TF/s err {err:.1e}")
print(" | ".join(out), flush=True)
