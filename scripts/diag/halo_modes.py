"""Halo conv time with parts switched off (conv debug flags: 1 no output stores, 2 no MMAs,
16384 no halo loads, 512 = the TMA-im2col path instead), B=256 ResNet-50 layer-1/2 3x3 shapes."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
for (N, Cin, H, W, Cout) in [(256, 64, 56, 56, 64), (256, 128, 28, 28, 128)]:
    d = L.ConvDesc(N, Cin, H, W, Cout, H, W, 3, 3, 1, 1, 1, 1, Cin, 1)
    x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
    w = torch.randn(Cout, Cin, 3, 3, device=dev) * 0.05
    b = torch.randn(Cout, device=dev)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
    y = torch.zeros(N, H, W, Cout, dtype=torch.bfloat16, device=dev)
    res = []
    outs = {}
    for dbg in (0, 1, 2, 3, 16384, 16385, 16386, 16387, 512):
        L.check(L.lib().sol_b200_set_conv_debug(dbg))
        for _ in range(3):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), b.data_ptr(), y.data_ptr(), 1, st))
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(20):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), b.data_ptr(), y.data_ptr(), 1, st))
        ev1.record()
        torch.cuda.synchronize()
        res.append(f"{dbg}:{ev0.elapsed_time(ev1) / 20 * 1e3:.1f}")
        if dbg in (0, 512):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), b.data_ptr(), y.data_ptr(), 1, st))
            torch.cuda.synchronize()
            outs[dbg] = y.clone()
    print((N, Cin, H, W, Cout), " ".join(res), flush=True)
    print("   halo == im2col:", torch.equal(outs[0], outs[512]),
          " max diff vs im2col:", (outs[0].float() - outs[512].float()).abs().max().item(), flush=True)
L.check(L.lib().sol_b200_set_conv_debug(0))
