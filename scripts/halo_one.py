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
L.check(L.lib().sol_b200_set_conv_debug(int(sys.argv[1]) if len(sys.argv) > 1 else 0))
for _ in range(3):
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
torch.cuda.synchronize(); print("ok")
