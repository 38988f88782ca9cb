"""Out-of-bounds access checks without compute-sanitizer (closed on this GPU pool): every operand
of a kernel lives inside a larger allocation whose surrounding guard bands hold sentinels --
NaN for inputs (a kernel reading past an operand poisons its output, caught by the finiteness
and parity checks) and a fixed byte pattern for outputs (a kernel writing past its output
changes the pattern). Covers the tcgen05 conv paths (fprop incl. halo / stem / TMA / im2col, dgrad
incl. sub-pixel classes, wgrad incl. split-K) on ragged shapes and every DFP unit family of the
test models, with the guard bands right against the operand bytes."""
import ctypes as C

import numpy as np
import pytest

from oracle import sol_oracle as O

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes of sentinel on each side
PATTERN = 0x5A


def _guarded(torch, nbytes, fill_nan, dev):
    """(base tensor, view of nbytes inside it at offset GUARD): guards NaN (bf16/f32 payload view
    decides) or PATTERN bytes."""
    total = nbytes + 2 * GUARD
    base = torch.full((total,), PATTERN, dtype=torch.uint8, device=dev)
    if fill_nan:
        base.view(torch.int16)[:] = 0x7FC0  # bf16 NaN; as f32 pairs it is NaN too (0x7FC07FC0)
    return base


def _check_guards(base, nbytes):
    b = base.cpu().numpy()
    head, tail = b[:GUARD], b[GUARD + nbytes:]
    return bool(np.all(head == PATTERN) and np.all(tail == PATTERN))


CASES = [
    # N, Cin, H, W, Cout, k, s, p
    (2, 64, 14, 14, 64, 3, 1, 1), (2, 64, 15, 15, 128, 3, 2, 1), (3, 128, 7, 7, 256, 1, 1, 0),
    (2, 256, 14, 14, 512, 1, 2, 0), (2, 3, 32, 32, 64, 7, 2, 3), (4, 64, 1, 1, 10, 1, 1, 0),
    (1, 32, 9, 9, 48, 3, 1, 1), (3, 64, 13, 29, 64, 3, 1, 1), (2, 512, 7, 7, 2048, 1, 1, 0),
    (5, 64, 11, 11, 256, 1, 1, 0),
]


def _pad8(c):
    return (c + 7) // 8 * 8


@pytest.mark.parametrize("case", CASES)
def test_conv_paths_stay_in_bounds(gpu, case):
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout, k, s, p = case
    OH, OW = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    cld, old = _pad8(Cin), _pad8(Cout)
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (N, H, W, Cin)).astype(np.float32)
    w = (rng.uniform(-1, 1, (Cout, Cin, k, k)) / np.sqrt(Cin * k * k)).astype(np.float32)
    dy = rng.uniform(-1, 1, (N, OH, OW, Cout)).astype(np.float32)

    def put(arr, ld):  # guarded bf16 NHWC operand, channel padding zeroed
        n = arr.shape[0] * arr.shape[1] * arr.shape[2] * ld * 2
        base = _guarded(torch, n, True, gpu)
        t = torch.zeros(arr.shape[:3] + (ld,), dtype=torch.float32)
        t[..., :arr.shape[3]] = torch.from_numpy(arr)
        base[GUARD:GUARD + n].view(torch.bfloat16)[:] = t.reshape(-1).to(torch.bfloat16).to(gpu)
        return base, base[GUARD:].data_ptr()

    xb, xp = put(x, cld)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, 1, old)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=gpu)
    wd = torch.from_numpy(w).to(gpu)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 0, st))
    ybytes = N * OH * OW * old * 2
    yb = _guarded(torch, ybytes, False, gpu)
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), xp, wp.data_ptr(), None, yb[GUARD:].data_ptr(), 1, st))
    torch.cuda.synchronize()
    assert _check_guards(yb, ybytes), "fprop wrote outside its output"
    y = yb[GUARD:GUARD + ybytes].view(torch.bfloat16).float().cpu().numpy().reshape(N, OH, OW, old)
    assert np.all(np.isfinite(y)), "fprop read outside its input (NaN guard reached the output)"
    want = O.conv2d(x.transpose(0, 3, 1, 2), w, None, (s, s), (p, p))
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()
    want = O.conv2d(bf(x.transpose(0, 3, 1, 2)), bf(w), None, (s, s), (p, p))
    assert O.oracle_err(y[..., :Cout].transpose(0, 3, 1, 2), want) <= 1e-2
    # wgrad (split-K workspace inside a guarded allocation too)
    dyb, dyp = put(dy, old)
    dw_bytes = Cout * Cin * k * k * 4
    dwb = _guarded(torch, dw_bytes, False, gpu)
    ws = C.c_uint64()
    dW = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, 1, old)
    L.check(L.lib().sol_b200_conv_wgrad_workspace(C.byref(dW), C.byref(ws)))
    wsb = _guarded(torch, max(int(ws.value), 16), False, gpu)
    if old == Cout:
        L.check(L.lib().sol_b200_conv_wgrad(C.byref(dW), dyp, xp, dwb[GUARD:].data_ptr(), wsb[GUARD:].data_ptr(), st))
        torch.cuda.synchronize()
        assert _check_guards(dwb, dw_bytes), "wgrad wrote outside dW"
        assert _check_guards(wsb, max(int(ws.value), 16)), "wgrad wrote outside its workspace"
        got = dwb[GUARD:GUARD + dw_bytes].view(torch.float32).cpu().numpy()
        assert np.all(np.isfinite(got)), "wgrad read outside its operands"
    # dgrad (channels multiple of 8 only)
    if Cin % 8 == 0 and Cout % 8 == 0:
        dD = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, 1)
        L.check(L.lib().sol_b200_conv_packed_elems(C.byref(dD), 1, C.byref(n)))
        wt = torch.zeros(n.value, dtype=torch.bfloat16, device=gpu)
        L.check(L.lib().sol_b200_conv_pack_weight(C.byref(dD), wd.data_ptr(), wt.data_ptr(), 1, st))
        dx_bytes = N * H * W * Cin * 2
        dxb = _guarded(torch, dx_bytes, False, gpu)
        L.check(L.lib().sol_b200_conv_dgrad(C.byref(dD), dyp, wt.data_ptr(), dxb[GUARD:].data_ptr(), st))
        torch.cuda.synchronize()
        assert _check_guards(dxb, dx_bytes), "dgrad wrote outside dx"
        dx = dxb[GUARD:GUARD + dx_bytes].view(torch.bfloat16).float().cpu().numpy()
        assert np.all(np.isfinite(dx)), "dgrad read outside its operands"
    del xb, dyb


@pytest.mark.parametrize("name", ["small_cnn", "resnet18", "resnet50", "densenet", "mobilenet"])
@pytest.mark.parametrize("train", [False, True], ids=["infer", "train"])
def test_dfp_and_heavy_units_stay_in_bounds(gpu, name, train):
    """Every unit of the test models through module_run with every operand in its own guarded
    allocation (inputs NaN-guarded, output pattern-guarded)."""
    import torch
    from paper_2003_10688_b200 import _lib as L
    from paper_2003_10688_b200.dfp import create_module, is_f32_tensor, storage_bytes
    from paper_2003_10688_b200.graph import Meta
    from tests.gpu_util import quant, to_device
    from tests.test_gpu_units import _compile, _inputs
    if name in ("densenet", "mobilenet") and train:
        pytest.skip("extension-op training graphs are covered by test_gpu_units")
    batch = 4
    gp, units = _compile(name, train, batch)
    env = O.run_graph(gp, _inputs(gp, batch, seed=2))
    st = torch.cuda.current_stream().cuda_stream
    bad = []
    for u in units:
        mod = create_module(gp, u, 1)
        keep, ptrs = [], []
        for nm in list(u.inputs) + list(u.params):
            if nm in gp.params:
                t = to_device(gp.params[nm], Meta("plain", gp.params[nm].shape), 1, gpu, True)
            else:
                t = to_device(quant(env[nm], 1), gp.meta_of(nm), 1, gpu, f32=is_f32_tensor(gp, nm))
            raw = t.reshape(-1).view(torch.uint8)
            base = _guarded(torch, raw.numel(), True, gpu)
            base[GUARD:GUARD + raw.numel()] = raw
            keep.append(base)
            ptrs.append(base[GUARD:].data_ptr())
        ob = storage_bytes(gp.meta_of(u.output), 1, is_f32_tensor(gp, u.output))
        out = _guarded(torch, ob, False, gpu)
        keep.append(out)
        ptrs.append(out[GUARD:].data_ptr())
        scratch = torch.zeros(max(16, mod.scratch_bytes // 4 + 16), dtype=torch.float32, device=gpu)
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        L.check(L.lib().sol_b200_module_run(mod.handle, arr, len(ptrs), C.c_void_p(scratch.data_ptr()),
                                            C.c_void_p(st), 0))
        torch.cuda.synchronize()
        L.lib().sol_b200_module_destroy(mod.handle)
        if not _check_guards(out, ob):
            bad.append((u.output, mod.family, "write outside output"))
        f32 = is_f32_tensor(gp, u.output)
        vals = out[GUARD:GUARD + ob].view(torch.float32 if f32 else torch.bfloat16).float().cpu().numpy()
        if not np.all(np.isfinite(vals)):
            bad.append((u.output, mod.family, "non-finite output (read outside an input?)"))
    assert not bad, bad
