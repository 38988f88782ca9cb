"""Time one conv shape under a list of conv debug flags (1 = skip stores, 2 = skip MMA,
512 = halo kernel, 1024 = no resident B): python scripts/conv_dbg.py N Cin H W Cout k s p dbg..."""
import ctypes as C
import sys

import torch

sys.path.insert(0, '.')
from paper_2003_10688_b200 import _lib as L  # noqa: E402


def main():
    N, Cin, H, W, Cout, k, s, p = (int(v) for v in sys.argv[1:9])
    dbgs = [int(v) for v in sys.argv[9:]] or [0]
    dev = torch.device("cuda:0")
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
    flops = 2.0 * N * OH * OW * Cout * Cin * k * k
    ref = None
    for dbg in dbgs:
        L.check(L.lib().sol_b200_set_conv_debug(dbg))
        for _ in range(3):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
        torch.cuda.synchronize()
        if dbg & 3 == 0:
            if ref is None:
                ref = y.float().clone()
            err = (y.float() - ref).abs().max().item()
        else:
            err = float("nan")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # a CUDA graph of the 20 launches: the timing is the device's, not the host launch path's
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            g.capture_begin()
            for _ in range(20):
                L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1,
                                                    s2.cuda_stream))
            g.capture_end()
        g.replay()
        torch.cuda.synchronize()
        import time
        h0 = time.perf_counter()
        for _ in range(20):
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), None, y.data_ptr(), 1, st))
        host_us = (time.perf_counter() - h0) / 20 * 1e6
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 50.0
        print(f"dbg {dbg:5d}: {us:8.1f} us  {flops / us / 1e6:7.1f} TF/s  maxdiff-vs-first {err:.3g}  host {host_us:.1f} us/launch", flush=True)
    L.check(L.lib().sol_b200_set_conv_debug(0))


if __name__ == "__main__":
    main()
