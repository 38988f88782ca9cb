"""Micro-benchmark of the tcgen05 weight-gradient kernel (plus its split-K reduction) on the
ResNet-50 training shapes (B=128): python scripts/wgrad_micro.py [name ...] [--ncu] (one launch each)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda:0")
SHAPES = [  # N, Cin, H, W, Cout, k, s, p, name
    (128, 64, 56, 56, 64, 3, 1, 1, "l1.conv2"),
    (128, 256, 56, 56, 64, 1, 1, 0, "l1.conv1"),
    (128, 64, 56, 56, 256, 1, 1, 0, "l1.conv3"),
    (128, 128, 28, 28, 128, 3, 1, 1, "l2.conv2"),
    (128, 256, 56, 56, 128, 1, 1, 0, "l2.0.conv1"),
    (128, 256, 14, 14, 256, 3, 1, 1, "l3.conv2"),
    (128, 1024, 14, 14, 256, 1, 1, 0, "l3.conv1"),
    (128, 512, 7, 7, 512, 3, 1, 1, "l4.conv2"),
    (128, 512, 7, 7, 2048, 1, 1, 0, "l4.conv3"),
    (128, 2048, 7, 7, 512, 1, 1, 0, "l4.conv1"),
]


def run(shape, reps=10, ncu=False):
    N, Cin, H, W, Cout, k, s, p, name = shape
    st = torch.cuda.current_stream().cuda_stream
    OH = (H + 2 * p - k) // s + 1
    OW = (W + 2 * p - k) // s + 1
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, 1)
    x = torch.randn(N, H, W, Cin, device=dev).to(torch.bfloat16)
    dy = torch.randn(N, OH, OW, Cout, device=dev).to(torch.bfloat16)
    ws = C.c_uint64()
    L.check(L.lib().sol_b200_conv_wgrad_workspace(C.byref(d), C.byref(ws)))
    wsd = torch.zeros(ws.value // 4 + 64, dtype=torch.float32, device=dev)
    dw = torch.empty(Cout, Cin, k, k, dtype=torch.float32, device=dev)

    def once():
        L.check(L.lib().sol_b200_conv_wgrad(C.byref(d), dy.data_ptr(), x.data_ptr(), dw.data_ptr(), wsd.data_ptr(), st))
    if ncu:
        once()
        torch.cuda.synchronize()
        return
    for _ in range(3):
        once()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000.0 / reps
    flops = 2.0 * N * OH * OW * Cout * Cin * k * k
    byts = (x.numel() + dy.numel()) * 2 + dw.numel() * 4
    sol = max(flops / 1416e12, byts / 6551e9) * 1e6
    print(f"{name:11s} {us:8.1f} us  {flops / us / 1e6:7.1f} TF/s  sol {sol:6.1f} us ({100 * sol / us:4.0f}%)  "
          f"workspace {ws.value / 1e6:6.1f} MB", flush=True)


if __name__ == "__main__":
    names = [a for a in sys.argv[1:] if not a.startswith("--")]
    for sh in SHAPES:
        if not names or sh[-1] in names:
            run(sh, ncu="--ncu" in sys.argv)
