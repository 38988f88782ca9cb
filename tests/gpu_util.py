"""Helpers for GPU parity tests: run one compiled unit module on oracle-supplied inputs
(the reference test pattern of proj/tests/test_dfp.cpp:26-45 `run_group`)."""
import ctypes as C

import numpy as np


def quant(a, dtype):
    """Round to the plan storage precision (bf16 RNE) — the precision the kernels read."""
    a = np.ascontiguousarray(a, np.float32)
    if dtype == 1:
        import torch
        return torch.from_numpy(a).to(torch.bfloat16).float().numpy()
    return a


def to_device(a, meta, dtype, dev, is_param=False, f32=False):
    import torch
    from paper_2003_10688_b200.dfp import storage_ld
    a = np.asarray(a, np.float32)
    if is_param or meta.kind in ("plain", "scalar"):
        return torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev)
    tdt = torch.float32 if (dtype == 0 or f32) else torch.bfloat16
    ld = storage_ld(meta, dtype)
    if meta.kind == "nchw":
        n, c, h, w = meta.shape
        t = torch.zeros((n, h, w, ld), dtype=torch.float32)
        t[..., :c] = torch.from_numpy(a.reshape(meta.shape).transpose(0, 2, 3, 1).copy())
    else:
        n, c = meta.shape
        t = torch.zeros((n, ld), dtype=torch.float32)
        t[:, :c] = torch.from_numpy(a.reshape(meta.shape))
    return t.to(dev).to(tdt).contiguous()


def from_device(t, meta):
    a = t.float().cpu().numpy()
    if meta.kind == "nchw":
        n, c, h, w = meta.shape
        return a.reshape(n, h, w, -1)[..., :c].transpose(0, 3, 1, 2)
    if meta.kind == "nc":
        n, c = meta.shape
        return a.reshape(n, -1)[:, :c]
    return a.reshape(meta.shape)


def run_unit(g, unit, env, dtype, dev):
    """Compile `unit` of graph `g` and run it on inputs taken from the oracle environment `env`."""
    import torch
    from paper_2003_10688_b200 import _lib as L
    from paper_2003_10688_b200.dfp import create_module, is_f32_tensor, storage_bytes
    from paper_2003_10688_b200.graph import Meta
    mod = create_module(g, unit, dtype)
    args = []
    for name in list(unit.inputs) + list(unit.params):
        if name in g.params:
            args.append(to_device(g.params[name], Meta("plain", g.params[name].shape), dtype, dev, True))
        else:
            meta = g.meta_of(name)
            args.append(to_device(quant(env[name], dtype), meta, dtype, dev, f32=is_f32_tensor(g, name)))
    ometa = g.meta_of(unit.output)
    of32 = is_f32_tensor(g, unit.output)
    nbytes = storage_bytes(ometa, dtype, of32)
    out = torch.zeros(nbytes // (4 if (dtype == 0 or of32) else 2),
                      dtype=torch.float32 if (dtype == 0 or of32) else torch.bfloat16, device=dev)
    args.append(out)
    scratch = torch.zeros(max(16, mod.scratch_bytes // 4 + 16), dtype=torch.float32, device=dev)
    ptrs = (C.c_void_p * len(args))(*[t.data_ptr() for t in args])
    st = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().sol_b200_module_run(mod.handle, ptrs, len(args), C.c_void_p(scratch.data_ptr()),
                                        C.c_void_p(st), 0))
    torch.cuda.synchronize()
    L.lib().sol_b200_module_destroy(mod.handle)
    return mod.family, from_device(out, ometa)
