"""tcgen05 implicit-GEMM kernels (fprop / dgrad / wgrad) through the raw C ABI entry points,
checked against the numpy f64 oracle restatement of the reference conv (reference.cpp:138-161,
:482-533). Tolerances: TF32 / bf16 tensor-core math -> max relative error (oracle_err metric,
floor 1% of scale) <= 1e-2 as stated by the north star, measured against the oracle applied to the
operands rounded to the tensor-core input precision (the remaining error is f32 accumulation order
plus the bf16 rounding of the stored output)."""
import ctypes as C

import numpy as np
import pytest

from oracle import sol_oracle as O

pytestmark = pytest.mark.gpu

CASES = [
    # N, Cin, H, W, Cout, k, s, p
    (2, 64, 14, 14, 64, 3, 1, 1),
    (2, 64, 15, 15, 128, 3, 2, 1),
    (3, 128, 7, 7, 256, 1, 1, 0),
    (2, 256, 14, 14, 512, 1, 2, 0),
    (2, 3, 32, 32, 64, 7, 2, 3),      # stem (channels padded to 16 bytes)
    (4, 64, 1, 1, 10, 1, 1, 0),       # linear-shaped, ragged N
    (1, 32, 9, 9, 48, 3, 1, 1),
    (16, 64, 28, 28, 64, 3, 1, 1),    # many pixel k-blocks: split wgrad (swapped orientation)
    (8, 64, 28, 28, 256, 1, 1, 0),
    (3, 64, 56, 56, 64, 3, 1, 1),     # halo-tile kernel (halo.cu), ResNet-50 layer-1 shape
    (2, 64, 13, 29, 64, 3, 1, 1),     # halo-tile kernel, ragged rows / junk columns
    (2, 128, 28, 28, 128, 3, 1, 1),   # ResNet-50 layer-2 shape: halo fprop, halo wgrad by filter row
    (3, 128, 11, 19, 128, 3, 1, 1),   # halo wgrad (128 channels), ragged rows / junk columns
    (2, 256, 14, 14, 256, 3, 1, 1),   # ResNet-50 layer 3: halo wgrad by (tap pair, ci slice)
    (2, 512, 7, 7, 512, 3, 1, 1),     # ResNet-50 layer 4: 64-row units, two co slices
    (1, 256, 9, 11, 512, 3, 1, 1),    # wide halo wgrad, ragged
    (1, 64, 5, 5, 64, 3, 1, 1),       # halo wgrad with a single unit (one partial, still reduced)
]


def quant(a, dt):
    """Operand precision of the tensor-core path: bf16 round-to-nearest-even, or TF32
    (f32 with the low 13 mantissa bits dropped)."""
    a = np.ascontiguousarray(a, np.float32)
    if dt == 1:
        import torch
        return torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def _pad_c(c, dt):
    v = 8 if dt == 1 else 4
    return (c + v - 1) // v * v


def _to_nhwc(torch, x, cld, dt, dev):
    n, c, h, w = x.shape
    t = torch.zeros((n, h, w, cld), dtype=torch.float32)
    t[..., :c] = torch.from_numpy(x.transpose(0, 2, 3, 1).copy())
    return t.to(dev).to(torch.bfloat16 if dt == 1 else torch.float32).contiguous()


@pytest.mark.parametrize("dt", [1, 0], ids=["bf16", "tf32"])
@pytest.mark.parametrize("case", CASES)
def test_conv_fprop(gpu, case, dt):
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout, k, s, p = case
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (N, Cin, H, W)).astype(np.float32)
    w = rng.uniform(-0.2, 0.2, (Cout, Cin, k, k)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, Cout).astype(np.float32)
    OH = (H + 2 * p - k) // s + 1
    OW = (W + 2 * p - k) // s + 1
    cld = _pad_c(Cin, dt)
    old = _pad_c(Cout, dt)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, dt, old)
    xd = _to_nhwc(torch, x, cld, dt, gpu)
    wd = torch.from_numpy(w).to(gpu)
    bd = torch.from_numpy(b).to(gpu)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=xd.dtype, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 0, st))
    y = torch.full((N, OH, OW, old), 7.0, dtype=xd.dtype, device=gpu)
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), xd.data_ptr(), wp.data_ptr(), bd.data_ptr(), y.data_ptr(), dt, st))
    torch.cuda.synchronize()
    yy = y.float().cpu().numpy()
    assert np.all(yy[..., Cout:] == 0.0)  # row padding is written as zeros
    got = yy[..., :Cout].transpose(0, 3, 1, 2)
    want = O.conv2d(quant(x, dt), quant(w, dt), b, (s, s), (p, p))
    err = O.oracle_err(got, want)
    assert err <= 1e-2, err


@pytest.mark.parametrize("dt", [1, 0], ids=["bf16", "tf32"])
@pytest.mark.parametrize("case", [c for c in CASES if c[1] % 8 == 0 and c[4] % 8 == 0])
def test_conv_dgrad(gpu, case, dt):
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout, k, s, p = case
    rng = np.random.default_rng(2)
    OH = (H + 2 * p - k) // s + 1
    OW = (W + 2 * p - k) // s + 1
    dy = rng.uniform(-1, 1, (N, Cout, OH, OW)).astype(np.float32)
    w = rng.uniform(-0.2, 0.2, (Cout, Cin, k, k)).astype(np.float32)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, dt)
    dyd = _to_nhwc(torch, dy, Cout, dt, gpu)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 1, C.byref(n)))
    wp = torch.zeros(n.value, dtype=dyd.dtype, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    wd = torch.from_numpy(w).to(gpu)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 1, st))
    dx = torch.zeros((N, H, W, Cin), dtype=dyd.dtype, device=gpu)
    L.check(L.lib().sol_b200_conv_dgrad(C.byref(d), dyd.data_ptr(), wp.data_ptr(), dx.data_ptr(), st))
    torch.cuda.synchronize()
    got = dx.float().cpu().numpy().transpose(0, 3, 1, 2)
    want = O.conv2d_back_x(quant(dy, dt), quant(w, dt), (H, W), (s, s), (p, p))
    err = O.oracle_err(got, want)
    assert err <= 1e-2, err


@pytest.mark.parametrize("dt", [1, 0], ids=["bf16", "tf32"])
@pytest.mark.parametrize("case", [c for c in CASES if c[4] % 8 == 0])
def test_conv_wgrad(gpu, case, dt):
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout, k, s, p = case
    rng = np.random.default_rng(3)
    OH = (H + 2 * p - k) // s + 1
    OW = (W + 2 * p - k) // s + 1
    dy = rng.uniform(-1, 1, (N, Cout, OH, OW)).astype(np.float32)
    x = rng.uniform(-1, 1, (N, Cin, H, W)).astype(np.float32)
    cld = _pad_c(Cin, dt)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, dt)
    dyd = _to_nhwc(torch, dy, Cout, dt, gpu)
    xd = _to_nhwc(torch, x, cld, dt, gpu)
    ws = C.c_uint64()
    L.check(L.lib().sol_b200_conv_wgrad_workspace(C.byref(d), C.byref(ws)))
    wsd = torch.zeros(ws.value // 4 + 64, dtype=torch.float32, device=gpu)
    dw = torch.zeros((Cout, Cin, k, k), dtype=torch.float32, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().sol_b200_conv_wgrad(C.byref(d), dyd.data_ptr(), xd.data_ptr(), dw.data_ptr(), wsd.data_ptr(), st))
    torch.cuda.synchronize()
    want = O.conv2d_back_w(quant(dy, dt), quant(x, dt), (k, k), (s, s), (p, p))
    err = O.oracle_err(dw.cpu().numpy(), want)
    assert err <= 1e-2, err


@pytest.mark.parametrize("case", [(3, 64, 56, 56, 64), (2, 64, 13, 29, 64), (2, 64, 14, 14, 40),
                                  (2, 128, 28, 28, 128), (2, 128, 13, 29, 96)])
def test_halo_conv_matches_im2col(gpu, case):
    """The row-padded halo-tile conv (halo.cu) accumulates the same k-blocks in the same order
    as the TMA-im2col kernel, so the two outputs are bit-identical (conv debug flag 512 turns the
    halo path off)."""
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout = case
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream().cuda_stream
    d = L.ConvDesc(N, Cin, H, W, Cout, H, W, 3, 3, 1, 1, 1, 1, Cin, 1)
    g = torch.Generator().manual_seed(3)
    x = (torch.rand(N, H, W, Cin, generator=g) * 2 - 1).to(dev).to(torch.bfloat16)
    w = ((torch.rand(Cout, Cin, 3, 3, generator=g) * 2 - 1) * 0.1).to(dev)
    bias = (torch.rand(Cout, generator=g) - 0.5).to(dev)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=dev)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), w.data_ptr(), wp.data_ptr(), 0, st))
    outs = []
    try:
        for dbg in (0, 512):
            L.check(L.lib().sol_b200_set_conv_debug(dbg))
            y = torch.full((N, H, W, Cout), float("nan"), dtype=torch.bfloat16, device=dev)
            L.check(L.lib().sol_b200_conv_fprop(C.byref(d), x.data_ptr(), wp.data_ptr(), C.c_void_p(bias.data_ptr()),
                                                y.data_ptr(), 1, st))
            torch.cuda.synchronize()
            outs.append(y.float().cpu())
    finally:
        L.check(L.lib().sol_b200_set_conv_debug(0))
    assert torch.equal(outs[0], outs[1])
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.to(torch.bfloat16).float(), bias, padding=1)
    err = (outs[0].permute(0, 3, 1, 2) - ref.cpu()).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item()
