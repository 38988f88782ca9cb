"""clock64 trace of block 0 of the halo conv (debug flag 64): per tile, the cycle at which the
MMA warp starts it and at which the epilogue receives it."""
import ctypes as C, sys, torch
sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L
dev = torch.device("cuda:0"); st = torch.cuda.current_stream().cuda_stream
N, Cin, H, W, Cout = 256, 64, 56, 56, 64
d = L.ConvDesc(N, Cin, H, W, Cout, H, W, 3, 3, 1, 1, 1, 1, Cin, 1)
x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
w = torch.randn(Cout, Cin, 3, 3, device=dev) * 0.05
n = C.c_int64(); L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
y = torch.zeros(N, H, W, Cout, dtype=torch.bfloat16, device=dev)
for dbg in [int(v) for v in sys.argv[1:]]:
    L.check(L.lib().sol_b200_set_conv_debug(dbg))
    for _ in range(2):
        L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
    torch.cuda.synchronize()
    ts = y.view(-1).view(torch.int64)[:384].cpu().numpy().reshape(6, 64)
    mma, epi = ts[1], ts[2]
    base = mma[0]
    print("   kernel start", int(ts[0, 0] - base), "weights resident", int(ts[0, 1] - base))
    for j in range(6):
        print("   tile", j, "top", int(ts[3, j] - base), "after tempty", int(ts[4, j] - base), "start", int(mma[j] - base),
              "loop done", int(ts[5, j] - base), "epi", int(epi[j] - base))
    base = mma[0]
    print("dbg", dbg, "mma start", [int(v - base) for v in mma[:12]])
    print("   epi", [int(v - base) for v in epi[:12]])
    print("   mma deltas", [int(mma[i + 1] - mma[i]) for i in range(40)])
