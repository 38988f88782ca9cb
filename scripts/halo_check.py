"""Halo conv kernel vs the generic im2col path on R50 3x3 shapes (both base-offset modes)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
for (N, Cin, H, W, Cout) in [(4, 64, 56, 56, 64), (4, 128, 28, 28, 128), (2, 64, 20, 20, 128), (256, 64, 56, 56, 64), (256, 128, 28, 28, 128)]:
    d = L.ConvDesc(N, Cin, H, W, Cout, H, W, 3, 3, 1, 1, 1, 1, Cin, 1)
    x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
    w = torch.randn(Cout, Cin, 3, 3, device=dev) * 0.05
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
    outs = {}
    for mode, dbg in (("im2col", 0), ("halo", 512), ("nostore", 513), ("nomma", 514), ("neither", 515)):
        y = torch.zeros(N, H, W, Cout, dtype=torch.bfloat16, device=dev)
        L.check(L.lib().sol_b200_set_conv_debug(dbg))
        L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(10):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
        ev1.record()
        torch.cuda.synchronize()
        outs[mode] = (y.float(), ev0.elapsed_time(ev1) / 10 * 1e3)
    ref = outs["im2col"][0]
    sc = ref.abs().max().item()
    print((N, Cin, H, W, Cout), " ".join(f"{k}: {t:7.1f} us err {(v - ref).abs().max().item() / sc:.2e}" for k, (v, t) in outs.items()))
L.check(L.lib().sol_b200_set_conv_debug(0))
