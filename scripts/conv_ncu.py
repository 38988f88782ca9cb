"""One fprop launch of a chosen ResNet-50 conv shape (B=256) for ncu captures:
python scripts/conv_ncu.py <name>  (names as in conv_micro.py)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402
from scripts.conv_micro import SHAPES  # noqa: E402

dev = torch.device("cuda:0")
name = sys.argv[1]
N, Cin, H, W, Cout, k, s, p, _ = next(sh for sh in SHAPES if sh[-1] == name)
st = torch.cuda.current_stream().cuda_stream
OH = (H + 2 * p - k) // s + 1
OW = (W + 2 * p - k) // s + 1
d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, 1)
x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
w = torch.randn(Cout, Cin, k, k, device=dev) * 0.05
n = C.c_int64()
L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
y = torch.empty(N, OH, OW, Cout, dtype=torch.bfloat16, device=dev)
for _ in range(3):
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
torch.cuda.synchronize()
print("ok", name)
