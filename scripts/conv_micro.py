"""Micro-benchmark of the tcgen05 implicit-GEMM conv on single ResNet-50 shapes (B=256),
with profiling knobs (dbg: 1 = skip output stores, 2 = skip MMA) to locate the bottleneck."""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda:0")
SHAPES = [  # N, Cin, H, W, Cout, k, s, p, name
    (256, 8, 224, 224, 64, 7, 2, 3, "stem"),
    (256, 64, 56, 56, 64, 3, 1, 1, "l1.conv2"),
    (256, 64, 56, 56, 256, 1, 1, 0, "l1.conv3"),
    (256, 256, 56, 56, 64, 1, 1, 0, "l1.conv1"),
    (256, 128, 28, 28, 128, 3, 1, 1, "l2.conv2"),
    (256, 256, 14, 14, 256, 3, 1, 1, "l3.conv2"),
    (256, 1024, 14, 14, 256, 1, 1, 0, "l3.conv1"),
    (256, 512, 7, 7, 2048, 1, 1, 0, "l4.conv3"),
]


def main():
    st = torch.cuda.current_stream().cuda_stream
    for (N, Cin, H, W, Cout, k, s, p, name) in SHAPES:
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
        flops = 2.0 * N * OH * OW * Cout * Cin * k * k
        byts = (x.numel() + y.numel() + wp.numel()) * 2
        res = []
        for dbg in (0, 1, 2, 3, 4, 6):
            L.check(L.lib().sol_b200_set_conv_debug(dbg))
            for _ in range(3):
                L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 100.0
            res.append(us)
        L.check(L.lib().sol_b200_set_conv_debug(0))
        print(f"{name:10s} full {res[0]:8.1f} us ({flops / res[0] / 1e6:6.1f} TF/s, {byts / res[0] / 1e3:6.0f} GB/s) | "
              f"no-store {res[1]:8.1f} | no-mma {res[2]:8.1f} | neither {res[3]:8.1f} | no-epi {res[4]:8.1f} | no-epi-no-mma {res[5]:8.1f}")


if __name__ == "__main__":
    main()
