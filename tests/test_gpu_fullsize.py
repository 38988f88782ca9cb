"""Full-size parity of exactly what bench.py times (VERDICT r1 "what's weak" #1).

* The inference plan bench.py builds (ResNet-50, 224x224, batch 256, bf16, fuse_epilogue, default
  dual-GEMM / halo / direct-NCHW-stem paths) is run through predict() and 16 of its images are
  compared against the REFERENCE's own compiled f32 CPU path (oracle/_ref `run_compiled`: the
  unmodified reference sources' partition -> lower_group/run_kernel + heuristic_choice/
  execute_choice), one image per host thread. Bars (north star): oracle_err <= 1e-2 on the
  probabilities, top-1 agreement on every image whose reference margin is clear of the band, and
  at least one such image (the check is never vacuous).
* Every ResNet-50 implicit-GEMM shape (SURVEY 8d, 23 conv shapes) through the raw C ABI at N=2:
  fprop, dgrad and wgrad against the numpy f64 oracle on bf16-rounded operands.
* The bottleneck dual GEMM at the widths the bench uses (Nout 1024 and 2048: the 256-wide
  single-accumulator variant) against the oracle and the unfused plan.
* The training plan bench.py times (ResNet-50 224, batch 128, bf16): the arena-packed plan is
  bit-identical to the same plan with every buffer kept (no arena reuse), and every distinct unit
  (op signature x shapes) of that kept plan is re-checked against the oracle on the plan's own
  input buffers (the reference test pattern proj/tests/test_dfp.cpp:26-45).
"""
import ctypes as C
import os
import threading

import numpy as np
import pytest

from oracle import sol_oracle as O

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _clear_rows(want, tol=TOL):
    """Rows whose reference top-1 beats the runner-up by more than 4x the error band."""
    srt = np.sort(want, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.maximum(np.abs(srt[:, -1]), 1e-12)
    return margin > 4 * tol


# ------------------------------------------------------------------------------------------------
# inference: the bench plan vs the reference's compiled CPU path
# ------------------------------------------------------------------------------------------------

def _reference_compiled(g, xs, threads):
    """prob of each image from oracle/_ref run_compiled (batch-1 sessions, eval BN)."""
    from oracle import refbridge
    from paper_2003_10688_b200 import graph
    if not refbridge.available():
        pytest.skip("oracle/_ref/libsolref.so not built")
    mj, wb = graph.model_to_json(g), graph.weights_to_bytes(g.params)
    out = [None] * len(xs)
    todo = list(range(len(xs)))
    lock = threading.Lock()
    errors = []

    def worker():
        try:
            s = refbridge.RefSession(mj, wb, 1)
            s.pipeline()
            while True:
                with lock:
                    if not todo:
                        return
                    i = todo.pop()
                s.set_input("x", xs[i][None])
                s.run_compiled()
                out[i] = s.get("prob")
        except Exception as e:  # surfaced below
            errors.append(e)

    ths = [threading.Thread(target=worker) for _ in range(max(1, min(threads, len(xs))))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    return np.stack(out)


@pytest.fixture(scope="module")
def bench_infer():
    from paper_2003_10688_b200 import frontend, models
    g = models.resnet(50, hw=224, classes=1000)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=256, dtype="bf16", fuse_epilogue=True))
    return g, m


def test_bench_inference_plan_matches_reference(gpu, bench_infer):
    g, m = bench_infer
    fams = {st.family for st in m.steps}
    # the paths the bench times are the ones under test
    assert any(len(u.node_ids) >= 5 for u in m.units), "dual-GEMM bottleneck tails not formed"
    assert "x" not in {st.output for st in m.steps if st.kind == "reorder"}, "direct NCHW stem not used"
    assert any(f.startswith("conv_stem") for f in fams), fams
    rng = np.random.default_rng(1234)  # bench.py's input distribution
    x = rng.uniform(-1, 1, (256, 3, 224, 224)).astype(np.float32)
    prob = m.predict({"x": x})["prob"]
    assert prob.shape == (256, 1000) and np.all(np.isfinite(prob))
    np.testing.assert_allclose(prob.sum(1), 1.0, rtol=1e-3)
    # 16 images spread over the batch (first, last and both CTA-tile boundary regions)
    idx = np.array([0, 1, 2, 63, 64, 100, 127, 128, 129, 170, 191, 200, 230, 253, 254, 255])
    want = _reference_compiled(g, x[idx], os.cpu_count() or 1)
    got = prob[idx]
    err = O.oracle_err(got, want)
    clear = _clear_rows(want)
    agree = np.argmax(got, 1) == np.argmax(want, 1)
    print(f"bench plan vs reference compiled path: oracle_err={err:.3e}, clear rows {int(clear.sum())}/16, "
          f"top-1 agreement {int(agree.sum())}/16")
    assert err <= TOL, err
    assert clear.sum() > 0, "no image has a clear reference top-1 margin: the top-1 check would be vacuous"
    assert np.all(agree[clear]), (np.argmax(got, 1), np.argmax(want, 1), clear)
    # CUDA-graph replay (what the bench times) gives the identical answer
    prob2 = m.predict({"x": x})["prob"]
    assert np.array_equal(prob, prob2)


# ------------------------------------------------------------------------------------------------
# every ResNet-50 conv shape through the raw ABI (N = 2)
# ------------------------------------------------------------------------------------------------

def _resnet50_conv_shapes(batch=2):
    from paper_2003_10688_b200 import graph, models
    g = graph.infer_shapes(models.resnet(50, hw=224, classes=1000), batch)
    seen = []
    for n in g.nodes:
        if n.op != "Conv2d":
            continue
        _, cin, h, w = g.meta_of(n.inputs[0]).shape
        a = n.attrs
        case = (batch, cin, h, w, a.out_channels, a.kh, a.sh, a.ph)
        if case not in seen:
            seen.append(case)
    return seen


R50 = _resnet50_conv_shapes()


def test_resnet50_has_23_conv_shapes():
    assert len(R50) == 23, R50


def _conv_case(case):
    import torch
    from paper_2003_10688_b200 import _lib as L
    N, Cin, H, W, Cout, k, s, p = case
    OH = (H + 2 * p - k) // s + 1
    OW = (W + 2 * p - k) // s + 1
    cld = (Cin + 7) // 8 * 8
    return torch, L, N, Cin, H, W, Cout, k, s, p, OH, OW, cld


def _nhwc(torch, x, cld, dev):
    n, c, h, w = x.shape
    t = torch.zeros((n, h, w, cld), dtype=torch.float32)
    t[..., :c] = torch.from_numpy(x.transpose(0, 2, 3, 1).copy())
    return t.to(dev).to(torch.bfloat16).contiguous()


@pytest.mark.parametrize("case", R50, ids=lambda c: "c{}-{}k{}s{}h{}".format(c[1], c[4], c[5], c[6], c[2]))
def test_resnet50_conv_fprop(gpu, case):
    torch, L, N, Cin, H, W, Cout, k, s, p, OH, OW, cld = _conv_case(case)
    rng = np.random.default_rng(11)
    x = rng.uniform(-1, 1, (N, Cin, H, W)).astype(np.float32)
    w = (rng.uniform(-1, 1, (Cout, Cin, k, k)) / np.sqrt(Cin * k * k)).astype(np.float32)
    b = rng.uniform(-0.5, 0.5, Cout).astype(np.float32)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, 1, Cout)
    xd = _nhwc(torch, x, cld, gpu)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 0, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    wd = torch.from_numpy(w).to(gpu)
    bd = torch.from_numpy(b).to(gpu)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 0, st))
    y = torch.full((N, OH, OW, Cout), float("nan"), dtype=torch.bfloat16, device=gpu)
    L.check(L.lib().sol_b200_conv_fprop(C.byref(d), xd.data_ptr(), wp.data_ptr(), bd.data_ptr(), y.data_ptr(), 1, st))
    torch.cuda.synchronize()
    got = y.float().cpu().numpy().transpose(0, 3, 1, 2)
    want = O.conv2d(_bf16(x), _bf16(w), b, (s, s), (p, p))
    err = O.oracle_err(got, want)
    assert np.all(np.isfinite(got)) and err <= TOL, err


@pytest.mark.parametrize("case", [c for c in R50 if c[1] % 8 == 0],
                         ids=lambda c: "c{}-{}k{}s{}h{}".format(c[1], c[4], c[5], c[6], c[2]))
def test_resnet50_conv_dgrad(gpu, case):
    torch, L, N, Cin, H, W, Cout, k, s, p, OH, OW, cld = _conv_case(case)
    rng = np.random.default_rng(12)
    dy = rng.uniform(-1, 1, (N, Cout, OH, OW)).astype(np.float32)
    w = (rng.uniform(-1, 1, (Cout, Cin, k, k)) / np.sqrt(Cout * k * k)).astype(np.float32)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, Cin, 1)
    dyd = _nhwc(torch, dy, Cout, gpu)
    n = C.c_int64()
    L.check(L.lib().sol_b200_conv_packed_elems(C.byref(d), 1, C.byref(n)))
    wp = torch.zeros(n.value, dtype=torch.bfloat16, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    wd = torch.from_numpy(w).to(gpu)
    L.check(L.lib().sol_b200_conv_pack_weight(C.byref(d), wd.data_ptr(), wp.data_ptr(), 1, st))
    dx = torch.full((N, H, W, Cin), float("nan"), dtype=torch.bfloat16, device=gpu)
    L.check(L.lib().sol_b200_conv_dgrad(C.byref(d), dyd.data_ptr(), wp.data_ptr(), dx.data_ptr(), st))
    torch.cuda.synchronize()
    got = dx.float().cpu().numpy().transpose(0, 3, 1, 2)
    want = O.conv2d_back_x(_bf16(dy), _bf16(w), (H, W), (s, s), (p, p))
    err = O.oracle_err(got, want)
    assert np.all(np.isfinite(got)) and err <= TOL, err


@pytest.mark.parametrize("case", R50, ids=lambda c: "c{}-{}k{}s{}h{}".format(c[1], c[4], c[5], c[6], c[2]))
def test_resnet50_conv_wgrad(gpu, case):
    torch, L, N, Cin, H, W, Cout, k, s, p, OH, OW, cld = _conv_case(case)
    rng = np.random.default_rng(13)
    dy = rng.uniform(-1, 1, (N, Cout, OH, OW)).astype(np.float32)
    x = rng.uniform(-1, 1, (N, Cin, H, W)).astype(np.float32)
    d = L.ConvDesc(N, Cin, H, W, Cout, OH, OW, k, k, s, s, p, p, cld, 1)
    dyd = _nhwc(torch, dy, Cout, gpu)
    xd = _nhwc(torch, x, cld, gpu)
    ws = C.c_uint64()
    L.check(L.lib().sol_b200_conv_wgrad_workspace(C.byref(d), C.byref(ws)))
    wsd = torch.zeros(ws.value // 4 + 64, dtype=torch.float32, device=gpu)
    dw = torch.full((Cout, Cin, k, k), float("nan"), dtype=torch.float32, device=gpu)
    st = torch.cuda.current_stream().cuda_stream
    L.check(L.lib().sol_b200_conv_wgrad(C.byref(d), dyd.data_ptr(), xd.data_ptr(), dw.data_ptr(), wsd.data_ptr(), st))
    torch.cuda.synchronize()
    want = O.conv2d_back_w(_bf16(dy), _bf16(x), (k, k), (s, s), (p, p))
    got = dw.cpu().numpy()
    err = O.oracle_err(got, want)
    assert np.all(np.isfinite(got)) and err <= TOL, err


# ------------------------------------------------------------------------------------------------
# the wide dual GEMM (bottleneck tail + downsample, Nout 1024 / 2048)
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cin,width,hw", [(512, 256, 28), (1024, 512, 14)], ids=["l3.0", "l4.0"])
def test_wide_dual_gemm_tail(gpu, cin, width, hw):
    from paper_2003_10688_b200 import frontend, graph
    from paper_2003_10688_b200.models import _bottleneck, _head
    from tests.test_gpu_units import _inputs
    b = graph.GraphBuilder(41)
    b.input("x", graph.meta_nchw(0, cin, hw, hw))
    y, cout = _bottleneck(b, "x", cin, width, 2, "blk")
    y = b.conv("tail", y, cout, 64, 1, 1, 0)  # a heavy consumer keeps the block's ReLU unit closed
    p = b.gap("gap", y)
    g = _head(b, p, 64, 10, False)
    batch = 8
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=17)
    fused = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True))
    dual = [u for u in fused.units if len(u.node_ids) >= 5]
    assert dual, "dual GEMM unit not formed"
    plain = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16"))
    got, ref = fused.predict(ins)["prob"], plain.predict(ins)["prob"]
    want = O.run_graph(gi, ins)["prob"]
    assert O.oracle_err(got, want) <= TOL
    assert O.oracle_err(got, ref) <= TOL
    # the dual unit's own output on the plan's own (bf16) inputs against the f64 oracle of the
    # folded GEMM the unit defines (pack.cu pack_dual_kernel: W' = bf16(W * gamma/sqrt(var+eps)) per
    # branch, one f32 bias of both shifted BN offsets): isolates the kernel from the (approximate,
    # end-to-end-checked above) BN fold, whose per-weight bf16 rounding the oracle_err metric's 1%
    # floor magnifies on near-zero outputs
    import torch
    from tests.gpu_util import from_device
    m1 = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True, keep_all=True))
    m1.predict(ins)

    def get(nm):
        raw = m1.read_tensor(nm)
        t = torch.from_numpy(raw.view(np.int16).copy()).view(torch.bfloat16)
        return from_device(t, m1.graph.meta_of(nm)).astype(np.float64)

    u = next(x for x in m1.units if len(x.node_ids) >= 5)
    nodes = [m1.graph.find_node(n) for n in u.node_ids]
    assert [n.op for n in nodes] == ["Conv2d", "BatchNorm2d", "Conv2d", "BatchNorm2d", "Add", "ReLU"]
    P = m1.params
    y = 0.0
    bias = np.zeros(nodes[0].attrs.out_channels)
    for conv, bn in ((nodes[0], nodes[1]), (nodes[2], nodes[3])):
        gam, bet, mean, var = (np.asarray(P[k], np.float64) for k in bn.params)
        sc = gam / np.sqrt(var + bn.attrs.eps)
        w = _bf16((P[conv.params[0]] * sc[:, None, None, None]).astype(np.float32)).astype(np.float64)
        cb = P[conv.params[1]] if (conv.attrs.has_bias and len(conv.params) > 1) else 0.0
        bias += (cb - mean) * sc + bet
        y = y + O.conv2d(get(conv.inputs[0]), w, None, (conv.attrs.sh, conv.attrs.sw), (0, 0))
    want = np.maximum(y + bias[None, :, None, None], 0.0)
    err = O.oracle_err(get(u.output), want)
    assert err <= TOL, err


# ------------------------------------------------------------------------------------------------
# training: the bench plan (ResNet-50 224, batch 128) -- arena vs keep-all, then per unit
# ------------------------------------------------------------------------------------------------

TRAIN_B = 128


@pytest.fixture(scope="module")
def bench_train():
    from paper_2003_10688_b200 import frontend, graph, models
    g = models.resnet(50, hw=224, classes=1000, train=True)
    rng = np.random.default_rng(1234)
    x = rng.uniform(-1, 1, (TRAIN_B, 3, 224, 224)).astype(np.float32)
    t = np.zeros((TRAIN_B, 1000), np.float32)
    t[np.arange(TRAIN_B), rng.integers(0, 1000, TRAIN_B)] = 1
    ins = {"x": x, "t": t}
    res = {}
    for keep in (False, True):
        m = frontend.optimize(g, frontend.OptimizeOptions(batch=TRAIN_B, dtype="bf16", train=True, lr=0.01,
                                                          keep_all=keep))
        loss = m.train_step(ins)
        res[keep] = (m, loss, m.gradients())
        if not keep:
            res["params_after"] = m.host_params()
    del graph
    return g, ins, res


def test_bench_train_plan_arena_is_bit_identical(gpu, bench_train):
    """Arena packing (transient buffers reused by liveness) must not change a single bit."""
    g, ins, res = bench_train
    (m0, l0, g0), (m1, l1, g1) = res[False], res[True]
    assert m0.arena_bytes() < m1.arena_bytes()
    assert np.isfinite(l0) and l0 == l1, (l0, l1)
    for k in g0:
        assert np.array_equal(g0[k], g1[k]), k
    new = res["params_after"]
    for k in list(g0)[:16]:
        np.testing.assert_allclose(new[k], g.params[k] - np.float32(0.01) * g0[k], rtol=1e-5, atol=1e-6)


# ops whose every output sample depends only on the same input sample (and no saved batch meta)
PER_SAMPLE = {"Conv2d", "Conv2dBackX", "ReLU", "ReLU6", "ReluBack", "Relu6Back", "MaxPool2d", "MaxPool2dBack",
              "AvgPool2d", "Add", "Copy", "GlobalAvgPool", "Flatten", "Linear", "LinearBackX", "Softmax"}


def test_bench_train_plan_units_match_oracle(gpu, bench_train):
    """One unit per distinct (op signature, input shapes) of the full-size training plan, re-run by
    the oracle on the plan's own input buffers (bf16-rounded weights for tensor-core units). Units
    whose ops are all per-sample are checked on the first 8 images; batch-coupled units (BatchNorm
    statistics / backward, weight gradients, the loss) on the whole batch."""
    import torch
    from paper_2003_10688_b200 import dfp
    from tests.gpu_util import from_device
    g, ins, res = bench_train
    m = res[True][0]

    def get(nm, rows=None):
        meta = m.graph.meta_of(nm)
        raw = m.read_tensor(nm)
        f32 = dfp.is_f32_tensor(m.graph, nm)
        t = torch.from_numpy(raw.view(np.float32).copy() if f32 else raw.view(np.int16).copy())
        a = from_device(t if f32 else t.view(torch.bfloat16), meta).astype(np.float64)
        return a[:rows] if (rows is not None and meta.kind in ("nchw", "nc")) else a

    seen, bad, checked = set(), [], 0
    for u in m.units:
        ops = tuple(m.graph.find_node(n).op for n in u.node_ids)
        key = (u.kind, ops, tuple(m.graph.meta_of(i).shape for i in u.inputs if i not in m.params))
        if key in seen:
            continue
        seen.add(key)
        rows = 8 if all(op in PER_SAMPLE for op in ops) else None
        params = {k: np.asarray(_bf16(v) if (u.kind == "dnn" and v.ndim >= 2) else v, np.float64)
                  for k, v in m.params.items()}
        local = {nm: get(nm, rows) for nm in u.inputs}
        for nid in u.node_ids:
            n = m.graph.find_node(nid)
            local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
        got = get(u.output, rows)
        err = O.oracle_err(got, local[u.output])
        if len(u.node_ids) == 3 and m.graph.find_node(u.node_ids[0]).op == "Conv2dBackX":
            # fused dgrad + Add + ReluBack (fusion.fuse_dgrad_relu_back; bit-identical to the unfused
            # plan): the sum of two gradients cancels, so one bf16 ulp of the rounded dgrad is
            # measured against the operands' magnitude, not the (possibly tiny) sum's
            add = m.graph.find_node(u.node_ids[1])
            mag = np.abs(local[add.inputs[0]]) + np.abs(local[add.inputs[1]])
            den = np.maximum(mag, max(0.01 * float(mag.max()), 1e-12))
            err = float(np.max(np.abs(got - local[u.output]) / den))
        checked += 1
        if not np.all(np.isfinite(got)) or err > 2e-2:
            bad.append((u.output, ops, err))
    print(f"full-size training plan: {checked} distinct units checked of {len(m.units)}")
    assert checked > 50
    assert not bad, bad


# ------------------------------------------------------------------------------------------------
# the other BASELINE configs at full size (bench.py other_configs): predict() on the full batch,
# images checked against the oracle (eval BatchNorm: images are independent)
# ------------------------------------------------------------------------------------------------

CONFIGS = [("small_cnn", 32, "f32", 32, 8), ("resnet18", 64, "f32", 224, 3),
           ("densenet121", 128, "bf16", 224, 2), ("mobilenet_v2", 128, "bf16", 224, 2)]


@pytest.mark.parametrize("model,batch,dtype,hw,check", CONFIGS, ids=[c[0] + "-" + c[2] for c in CONFIGS])
def test_baseline_config_full_size(gpu, model, batch, dtype, hw, check):
    """ResNet-18 f32/TF32 B=64 and the small CNN against the REFERENCE's compiled path; DenseNet-121
    and MobileNet-V2 (Concat / ReLU6: not in the reference IR, parity unpinned) against the numpy
    oracle restatement. Bars: oracle_err <= 1e-2 on the probabilities (TF32 / bf16 tensor cores),
    top-1 agreement on every clear row and at least one clear row."""
    from paper_2003_10688_b200 import frontend, graph, models
    g = models.MODELS[model](hw=hw) if model == "small_cnn" else models.MODELS[model]()
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype=dtype, fuse_epilogue=True, cache=False))
    x = np.random.default_rng(7).uniform(-1, 1, (batch, 3, hw, hw)).astype(np.float32)
    prob = m.predict({"x": x})["prob"]
    assert np.all(np.isfinite(prob))
    idx = np.linspace(0, batch - 1, check).astype(int)
    if model in ("small_cnn", "resnet18"):
        want = _reference_compiled(g, x[idx], os.cpu_count() or 1)
    else:
        want = O.run_graph(graph.infer_shapes(g, len(idx)), {"x": x[idx]})["prob"]
    got = prob[idx]
    err = O.oracle_err(got, want)
    clear = _clear_rows(want)
    print(f"{model} {dtype} B={batch}: oracle_err {err:.3e}, clear rows {int(clear.sum())}/{len(idx)}")
    assert err <= TOL, err
    assert clear.sum() > 0
    assert np.all(np.argmax(got, 1)[clear] == np.argmax(want, 1)[clear])
