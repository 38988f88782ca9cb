"""TEST INFRASTRUCTURE ONLY — CPU oracle (numpy, f64 accumulation, f32 storage between layers).

A restatement of the reference's naive per-layer interpreter
/root/reference/proj/src/reference.cpp (reference_node :130-587, run_reference :589-605) in
canonical NCHW layout, plus the reference's comparison metric oracle_err (src/tensor.cpp:324-329).
It is pinned against outputs of the reference itself (oracle/_ref/libsolref.so, built from the
reference sources by oracle/Makefile) through the committed fixtures in tests/golden/ and the
live cross-checks in tests/test_oracle.py.

Extensions the reference IR lacks (Concat along C0, ReLU6 and their gradients) are restated here
in the same style; their parity is UNPINNED (no reference implementation exists to check against).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg may use this
module, and only as the checker. The product package never imports it.
"""
from __future__ import annotations

from typing import Dict

import numpy as np


# ------------------------------------------------------------------------------------------------
# metrics (src/tensor.cpp:302-329)
# ------------------------------------------------------------------------------------------------

def max_rel_err(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-8)
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


def oracle_err(a, b) -> float:
    """Like max_rel_err but elements below 1% of the tensor scale are measured against that floor."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if a.size == 0:
        return 0.0
    scale = max(np.max(np.abs(a)), np.max(np.abs(b)))
    floor = max(0.01 * scale, 1e-8)
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), floor)
    return float(np.max(np.abs(a - b) / den))


# ------------------------------------------------------------------------------------------------
# forward ops (reference.cpp:138-291)
# ------------------------------------------------------------------------------------------------

def _pad(x, ph, pw, value=0.0):
    return np.pad(x, ((0, 0), (0, 0), (ph, ph), (pw, pw)), constant_values=value)


def conv2d(x, w, b=None, stride=(1, 1), pad=(0, 0), groups=1):
    """reference.cpp:138-161: y = b + sum x[n, g*icg+ic, oh*sh-ph+kh, ow*sw-pw+kw] * W[oc, ic, kh, kw]."""
    x = np.asarray(x, np.float64)
    w = np.asarray(w, np.float64)
    N, Cin, H, W = x.shape
    Cout, icg, KH, KW = w.shape
    sh, sw = stride
    ph, pw = pad
    OH = (H + 2 * ph - KH) // sh + 1
    OW = (W + 2 * pw - KW) // sw + 1
    xp = _pad(x, ph, pw)
    ocg = Cout // groups
    y = np.zeros((N, Cout, OH, OW))
    for g in range(groups):
        xs = xp[:, g * icg:(g + 1) * icg]
        wg = w[g * ocg:(g + 1) * ocg]
        for kh in range(KH):
            for kw in range(KW):
                patch = xs[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
                y[:, g * ocg:(g + 1) * ocg] += np.einsum("nchw,oc->nohw", patch, wg[:, :, kh, kw], optimize=True)
    if b is not None:
        y += np.asarray(b, np.float64)[None, :, None, None]
    return y


def linear(x, w, b=None):
    """reference.cpp:162-173."""
    y = np.asarray(x, np.float64) @ np.asarray(w, np.float64).T
    if b is not None:
        y = y + np.asarray(b, np.float64)[None, :]
    return y


def relu(x):
    x = np.asarray(x, np.float64)
    return np.where(x > 0, x, 0.0)


def relu6(x):
    return np.minimum(relu(x), 6.0)


def maxpool(x, k, stride, pad, min_init=-np.inf):
    """reference.cpp:178-195: max over in-bounds window taps, initialised with min_init."""
    x = np.asarray(x, np.float64)
    N, C, H, W = x.shape
    (KH, KW), (sh, sw), (ph, pw) = k, stride, pad
    OH = (H + 2 * ph - KH) // sh + 1
    OW = (W + 2 * pw - KW) // sw + 1
    xp = _pad(x, ph, pw, -np.inf)
    y = np.full((N, C, OH, OW), float(min_init))
    for kh in range(KH):
        for kw in range(KW):
            y = np.maximum(y, xp[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw])
    return y


def avgpool(x, k, stride, pad, count_padding=False):
    """reference.cpp:196-215: sum / (count_padding ? kh*kw : in-bounds count)."""
    x = np.asarray(x, np.float64)
    N, C, H, W = x.shape
    (KH, KW), (sh, sw), (ph, pw) = k, stride, pad
    OH = (H + 2 * ph - KH) // sh + 1
    OW = (W + 2 * pw - KW) // sw + 1
    xp = _pad(x, ph, pw)
    ones = _pad(np.ones((1, 1, H, W)), ph, pw)
    s = np.zeros((N, C, OH, OW))
    cnt = np.zeros((1, 1, OH, OW))
    for kh in range(KH):
        for kw in range(KW):
            s += xp[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
            cnt += ones[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
    return s / (KH * KW if count_padding else cnt)


def batch_stats(x):
    """reference.cpp:95-116: per-channel mean and biased variance over (N, H, W)."""
    x = np.asarray(x, np.float64)
    axes = (0, 2, 3) if x.ndim == 4 else (0,)
    mean = x.mean(axis=axes)
    var = ((x - _bc(mean, x)) ** 2).mean(axis=axes)
    return mean, var


def _bc(v, x):
    v = np.asarray(v, np.float64)
    return v[None, :, None, None] if x.ndim == 4 else v[None, :]


def batchnorm(x, gamma, beta, mean, var, eps=1e-5, training=False):
    """reference.cpp:216-237."""
    x = np.asarray(x, np.float64)
    if training:
        mean, var = batch_stats(x)
    rstd = 1.0 / np.sqrt(np.asarray(var, np.float64) + eps)
    return _bc(gamma, x) * (x - _bc(mean, x)) * _bc(rstd, x) + _bc(beta, x)


def gap(x):
    return np.asarray(x, np.float64).mean(axis=(2, 3))


def flatten(x):
    """reference.cpp:245-254: canonical row-major order over non-batch dims."""
    x = np.asarray(x, np.float64)
    return x.reshape(x.shape[0], -1)


def softmax(x):
    x = np.asarray(x, np.float64)
    m = x.max(axis=1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=1, keepdims=True)


def cross_entropy(p, t):
    """reference.cpp:278-291: -sum(t * log p) / B."""
    p = np.asarray(p, np.float64)
    t = np.asarray(t, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        v = np.where(t != 0, t * np.log(p), 0.0)
    return np.array(-v.sum() / p.shape[0])


# ------------------------------------------------------------------------------------------------
# backward ops (reference.cpp:294-584)
# ------------------------------------------------------------------------------------------------

def relu_back(delta, x):
    return np.where(np.asarray(x) > 0, np.asarray(delta, np.float64), 0.0)


def relu6_back(delta, x):
    x = np.asarray(x)
    return np.where((x > 0) & (x < 6), np.asarray(delta, np.float64), 0.0)


def maxpool_back(delta, x, k, stride, pad, min_init=-np.inf):
    """reference.cpp:301-327: route to the first max in (kh, kw) scan order, only if > min_init."""
    delta = np.asarray(delta, np.float64)
    x = np.asarray(x, np.float64)
    N, C, H, W = x.shape
    (KH, KW), (sh, sw), (ph, pw) = k, stride, pad
    OH, OW = delta.shape[2], delta.shape[3]
    xp = _pad(x, ph, pw, -np.inf)
    best = np.full((N, C, OH, OW), -np.inf)
    arg = np.full((N, C, OH, OW), -1, dtype=np.int64)
    for kh in range(KH):
        for kw in range(KW):
            v = xp[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
            upd = v > best
            best = np.where(upd, v, best)
            arg = np.where(upd, kh * KW + kw, arg)
    dxp = np.zeros((N, C, H + 2 * ph, W + 2 * pw))
    route = (arg >= 0) & (best > min_init)
    for kh in range(KH):
        for kw in range(KW):
            sel = route & (arg == kh * KW + kw)
            dxp[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw] += np.where(sel, delta, 0.0)
    return dxp[:, :, ph:ph + H, pw:pw + W]


def avgpool_back(delta, in_shape, k, stride, pad, count_padding=False):
    delta = np.asarray(delta, np.float64)
    N, C, H, W = in_shape
    (KH, KW), (sh, sw), (ph, pw) = k, stride, pad
    OH, OW = delta.shape[2], delta.shape[3]
    ones = _pad(np.ones((1, 1, H, W)), ph, pw)
    cnt = np.zeros((1, 1, OH, OW))
    for kh in range(KH):
        for kw in range(KW):
            cnt += ones[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
    share = delta / (KH * KW if count_padding else cnt)
    dxp = np.zeros((N, C, H + 2 * ph, W + 2 * pw))
    for kh in range(KH):
        for kw in range(KW):
            dxp[:, :, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw] += share
    return dxp[:, :, ph:ph + H, pw:pw + W]


def gap_back(delta, in_shape):
    N, C, H, W = in_shape
    return np.broadcast_to(np.asarray(delta, np.float64)[:, :, None, None] / (H * W), in_shape).copy()


def softmax_back(delta, y):
    delta = np.asarray(delta, np.float64)
    y = np.asarray(y, np.float64)
    dot = (delta * y).sum(axis=1, keepdims=True)
    return y * (delta - dot)


def softmax_ce_back(p, t):
    p = np.asarray(p, np.float64)
    return (p - np.asarray(t, np.float64)) / p.shape[0]


def ce_back(p, t):
    p = np.asarray(p, np.float64)
    return -np.asarray(t, np.float64) / (p * p.shape[0])


def bn_back_x(delta, x, gamma, eps=1e-5, training=True, var=None):
    """reference.cpp:382-430."""
    delta = np.asarray(delta, np.float64)
    x = np.asarray(x, np.float64)
    if not training:
        return _bc(gamma, x) * _bc(1.0 / np.sqrt(np.asarray(var, np.float64) + eps), x) * delta
    mean, v = batch_stats(x)
    rstd = 1.0 / np.sqrt(v + eps)
    axes = (0, 2, 3) if x.ndim == 4 else (0,)
    m = x.size / x.shape[1]
    xhat = (x - _bc(mean, x)) * _bc(rstd, x)
    dsum = delta.sum(axis=axes)
    dxhat = (delta * xhat).sum(axis=axes)
    return _bc(gamma, x) * _bc(rstd, x) * (delta - _bc(dsum / m, x) - xhat * _bc(dxhat / m, x))


def bn_back_gamma(delta, x, eps=1e-5, training=True, mean=None, var=None):
    delta = np.asarray(delta, np.float64)
    x = np.asarray(x, np.float64)
    if training:
        mean, var = batch_stats(x)
    rstd = 1.0 / np.sqrt(np.asarray(var, np.float64) + eps)
    axes = (0, 2, 3) if x.ndim == 4 else (0,)
    return (delta * (x - _bc(mean, x)) * _bc(rstd, x)).sum(axis=axes)


def bn_back_beta(delta):
    delta = np.asarray(delta, np.float64)
    return delta.sum(axis=(0, 2, 3) if delta.ndim == 4 else (0,))


def conv2d_back_x(delta, w, in_hw, stride=(1, 1), pad=(0, 0), groups=1):
    """reference.cpp:482-506: dx[ih] = sum delta[(ih+ph-kh)/sh] W[., ., kh] over divisible taps."""
    delta = np.asarray(delta, np.float64)
    w = np.asarray(w, np.float64)
    N, Cout, OH, OW = delta.shape
    _, icg, KH, KW = w.shape
    H, W = in_hw
    sh, sw = stride
    ph, pw = pad
    Cin = icg * groups
    ocg = Cout // groups
    Hp = max(H + 2 * ph, sh * (OH - 1) + KH)
    Wp = max(W + 2 * pw, sw * (OW - 1) + KW)
    dxp = np.zeros((N, Cin, Hp, Wp))
    for g in range(groups):
        dg = delta[:, g * ocg:(g + 1) * ocg]
        wg = w[g * ocg:(g + 1) * ocg]
        for kh in range(KH):
            for kw in range(KW):
                dxp[:, g * icg:(g + 1) * icg, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw] += \
                    np.einsum("nohw,oc->nchw", dg, wg[:, :, kh, kw], optimize=True)
    return dxp[:, :, ph:ph + H, pw:pw + W]


def conv2d_back_w(delta, x, k, stride=(1, 1), pad=(0, 0), groups=1):
    """reference.cpp:507-533."""
    delta = np.asarray(delta, np.float64)
    x = np.asarray(x, np.float64)
    N, Cout, OH, OW = delta.shape
    Cin = x.shape[1]
    KH, KW = k
    sh, sw = stride
    ph, pw = pad
    icg = Cin // groups
    ocg = Cout // groups
    xp = _pad(x, ph, pw)
    dw = np.zeros((Cout, icg, KH, KW))
    for g in range(groups):
        for kh in range(KH):
            for kw in range(KW):
                patch = xp[:, g * icg:(g + 1) * icg, kh:kh + sh * (OH - 1) + 1:sh, kw:kw + sw * (OW - 1) + 1:sw]
                dw[g * ocg:(g + 1) * ocg, :, kh, kw] = np.einsum(
                    "nohw,nchw->oc", delta[:, g * ocg:(g + 1) * ocg], patch, optimize=True)
    return dw


def conv2d_back_b(delta):
    return np.asarray(delta, np.float64).sum(axis=(0, 2, 3))


def linear_back_x(delta, w):
    return np.asarray(delta, np.float64) @ np.asarray(w, np.float64)


def linear_back_w(delta, x):
    return np.asarray(delta, np.float64).T @ np.asarray(x, np.float64)


def linear_back_b(delta):
    return np.asarray(delta, np.float64).sum(axis=0)


# ------------------------------------------------------------------------------------------------
# graph runner (reference.cpp:589-612) over paper_2003_10688_b200.graph.ModelGraph
# ------------------------------------------------------------------------------------------------

def eval_node(n, ins, params, g=None):
    a = n.attrs
    op = n.op
    k = (a.kh, a.kw)
    s = (a.sh, a.sw)
    p = (a.ph, a.pw)
    P = [params[q] for q in n.params]
    if op == "Conv2d":
        return conv2d(ins[0], P[0], P[1] if a.has_bias else None, s, p, a.groups)
    if op == "Linear":
        return linear(ins[0], P[0], P[1] if a.has_bias else None)
    if op == "ReLU":
        return relu(ins[0])
    if op == "ReLU6":
        return relu6(ins[0])
    if op == "Copy":
        return np.asarray(ins[0], np.float64)
    if op == "MaxPool2d":
        return maxpool(ins[0], k, s, p, a.min_init)
    if op == "AvgPool2d":
        return avgpool(ins[0], k, s, p, a.count_padding)
    if op == "BatchNorm2d":
        return batchnorm(ins[0], P[0], P[1], P[2], P[3], a.eps, a.training)
    if op == "Add":
        return np.asarray(ins[0], np.float64) + np.asarray(ins[1], np.float64)
    if op == "Concat":
        return np.concatenate([np.asarray(t, np.float64) for t in ins], axis=1)
    if op == "Flatten":
        return flatten(ins[0])
    if op == "GlobalAvgPool":
        return gap(ins[0])
    if op == "Softmax":
        return softmax(ins[0])
    if op == "CrossEntropyLoss":
        return cross_entropy(ins[0], ins[1])
    if op == "ReluBack":
        return relu_back(ins[0], ins[1])
    if op == "ReLU6Back":
        return relu6_back(ins[0], ins[1])
    if op == "MaxPool2dBack":
        return maxpool_back(ins[0], ins[1], k, s, p, a.min_init)
    if op == "AvgPool2dBack":
        return avgpool_back(ins[0], n.saved_meta.shape, k, s, p, a.count_padding)
    if op == "GlobalAvgPoolBack":
        return gap_back(ins[0], n.saved_meta.shape)
    if op == "FlattenBack":
        return np.asarray(ins[0], np.float64).reshape(n.saved_meta.shape)
    if op == "ConcatBack":
        c = n.saved_meta.shape[1]
        return np.asarray(ins[0], np.float64)[:, a.offset:a.offset + c]
    if op == "SoftmaxBack":
        return softmax_back(ins[0], ins[1])
    if op == "SoftmaxCeBack":
        return softmax_ce_back(ins[0], ins[1])
    if op == "CeBack":
        return ce_back(ins[0], ins[1])
    if op == "BatchNormBackX":
        if a.training:
            return bn_back_x(ins[0], ins[1], P[0], a.eps, True)
        return bn_back_x(ins[0], ins[1], P[0], a.eps, False, P[2])
    if op == "BatchNormBackGamma":
        if a.training:
            return bn_back_gamma(ins[0], ins[1], a.eps, True)
        return bn_back_gamma(ins[0], ins[1], a.eps, False, P[0], P[1])
    if op == "BatchNormBackBeta":
        return bn_back_beta(ins[0])
    if op == "Conv2dBackX":
        sm = n.saved_meta.shape
        return conv2d_back_x(ins[0], P[0], (sm[2], sm[3]), s, p, a.groups)
    if op == "Conv2dBackW":
        return conv2d_back_w(ins[0], ins[1], k, s, p, a.groups)
    if op == "Conv2dBackB":
        return conv2d_back_b(ins[0])
    if op == "LinearBackX":
        return linear_back_x(ins[0], P[0])
    if op == "LinearBackW":
        return linear_back_w(ins[0], ins[1])
    if op == "LinearBackB":
        return linear_back_b(ins[0])
    if op == "SgdUpdate":
        return np.asarray(ins[0], np.float64) - float(np.float32(a.lr)) * np.asarray(ins[1], np.float64)
    raise NotImplementedError(op)


def run_graph(g, inputs: Dict[str, np.ndarray], store_f32: bool = True) -> Dict[str, np.ndarray]:
    """Every node output in topological order; f64 accumulation, f32 storage between layers."""
    env = {}
    for gi in g.graph_inputs:
        v = np.asarray(inputs[gi.name], np.float64)
        env[gi.name] = v.astype(np.float32).astype(np.float64) if store_f32 else v
    params = {k: np.asarray(v, np.float64) for k, v in g.params.items()}
    for n in g.nodes:
        out = eval_node(n, [env[i] for i in n.inputs], params, g)
        env[n.id] = np.asarray(out, np.float32).astype(np.float64) if store_f32 else np.asarray(out)
    return env


def update_bn_running_stats(g, params: Dict[str, np.ndarray], env: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
    """autodiff.cpp:356-384: for every training BatchNorm2d, running_mean <- (1-m) rm + m mean and
    running_var <- (1-m) rv + m var_biased * count/(count-1), statistics of the BN input in f64 over
    all non-channel positions. Returns the updated parameter dict (inputs untouched)."""
    out = dict(params)
    for n in g.nodes:
        if n.op != "BatchNorm2d" or not n.attrs.training:
            continue
        x = np.asarray(env[n.inputs[0]], np.float64)
        axes = (0,) + tuple(range(2, x.ndim))
        count = x.size // x.shape[1]
        mean = x.mean(axis=axes)
        var = ((x - mean.reshape((1, -1) + (1,) * (x.ndim - 2))) ** 2).sum(axis=axes)
        unbias = count / (count - 1) if count > 1 else 1.0
        mom = n.attrs.momentum
        rm, rv = n.params[2], n.params[3]
        out[rm] = ((1 - mom) * np.asarray(params[rm], np.float64) + mom * mean).astype(np.float32)
        out[rv] = ((1 - mom) * np.asarray(params[rv], np.float64) + mom * (var / count) * unbias).astype(np.float32)
    return out
