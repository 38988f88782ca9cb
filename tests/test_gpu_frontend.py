"""The network API over the B200 backend (fe::OptimizedModel, include/sol/frontend.hpp:104-180):
train modes, runtime learning rate, parameter contexts, the compiled-model cache, CompileSummary,
autotune with a persistent TuneCache, and deployment bundles."""
import numpy as np
import pytest

from oracle import sol_oracle as O
from tests.test_gpu_units import _inputs

pytestmark = pytest.mark.gpu


def _model(train, seed=11):
    from paper_2003_10688_b200 import models
    return models.resnet(18, hw=32, classes=16, width=16, train=train, seed=seed)


def _opts(**kw):
    from paper_2003_10688_b200 import frontend
    kw.setdefault("batch", 8)
    kw.setdefault("dtype", "bf16")
    kw.setdefault("cache", False)
    return frontend.OptimizeOptions(**kw)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_transparent_and_native_steps_agree(gpu, dtype):
    """TrainMode::Transparent (gradients to the host, host SGD in f32, autodiff.cpp:331-354) and
    TrainMode::Native (SGD on the device) take the same step from the same state."""
    from paper_2003_10688_b200 import frontend, graph
    g = _model(True)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=3)
    a = frontend.optimize(g, _opts(dtype=dtype, train=True, lr=0.05))
    b = frontend.optimize(g, _opts(dtype=dtype, train=True, lr=0.05))
    la = a.train_step(ins, lr=0.02, mode=frontend.TrainMode.NATIVE)
    ga = a.gradients()
    lb = b.train_step(ins, lr=0.02, mode=frontend.TrainMode.TRANSPARENT)
    gb = b.gradients()
    assert la == lb
    pa, pb = a.host_params(), b.host_params()
    for k in pa:
        if k in ga:
            assert np.array_equal(ga[k], gb[k]), k
        np.testing.assert_allclose(pa[k], pb[k], rtol=1e-6, atol=1e-7, err_msg=k)
    for k, gr in ga.items():  # theta' = theta - lr * g, lr taken per call (not the compile-time 0.05)
        np.testing.assert_allclose(pa[k], g.params[k] - np.float32(0.02) * gr, rtol=1e-5, atol=1e-6, err_msg=k)
    # a second transparent step starts from the host-updated parameters on the device
    lb2 = b.train_step(ins, lr=0.02, mode=frontend.TrainMode.TRANSPARENT)
    la2 = a.train_step(ins, lr=0.02)
    # (the device SGD is one fused multiply-add, the host one rounds twice: ULP-level parameter
    # differences, which a bf16 forward pass turns into ~1e-4 loss differences)
    np.testing.assert_allclose(la2, lb2, rtol=2e-3)


def test_runtime_learning_rate_zero_is_identity(gpu):
    from paper_2003_10688_b200 import frontend, graph
    g = _model(True)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=4)
    m = frontend.optimize(g, _opts(train=True, lr=0.1))
    m.train_step(ins, lr=0.0)
    new = m.host_params()
    for k, v in g.params.items():
        if not k.endswith(("running_mean", "running_var")):
            assert np.array_equal(new[k], v), k


def test_parameter_contexts_follow_training(gpu):
    """predict() on a training model runs its forward plan, re-synchronised with the trained
    parameters (sync_host_params + ensure_context); it equals a fresh inference model loaded
    with the same parameters bit for bit."""
    from paper_2003_10688_b200 import frontend, graph
    g = _model(True)
    gi = _model(False)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=5)
    x = {"x": ins["x"]}
    m = frontend.optimize(g, _opts(train=True, lr=0.05))
    p0 = m.predict(x)["prob"]
    ref0 = frontend.optimize(gi, _opts()).predict(x)["prob"]
    assert np.array_equal(p0, ref0)
    v0 = m.param_version
    for _ in range(2):
        m.train_step(ins)
    assert m.param_version == v0 + 2
    p1 = m.predict(x)["prob"]
    assert not np.array_equal(p0, p1)
    fresh = frontend.optimize(gi, _opts())
    fresh.load_state(m.host_params())
    assert np.array_equal(p1, fresh.predict(x)["prob"])
    # load_state invalidates every context: back to the initial parameters
    m.load_state(g.params)
    assert np.array_equal(m.predict(x)["prob"], p0)


def test_compile_cache_and_summary(gpu):
    from paper_2003_10688_b200 import frontend, graph
    g = _model(False)
    a = frontend.optimize(g, _opts(cache=True))
    assert not a.summary.cached and a.summary.units == len(a.units) > 0
    assert a.summary.dfp_units + a.summary.dnn_units == a.summary.units and a.summary.kernels >= a.summary.units
    b = frontend.optimize(_model(False), _opts(cache=True))
    assert b is a and b.summary.cached
    c = frontend.optimize(g, _opts(cache=True, fuse_epilogue=True))
    assert c is not a
    # same structure, other weights: the cached model with the new weights loaded
    g2 = _model(False, seed=12)
    d = frontend.optimize(g2, _opts(cache=True))
    assert d is a
    x = _inputs(graph.infer_shapes(g2, 8), 8, seed=6)
    want = frontend.optimize(g2, _opts()).predict(x)["prob"]
    assert np.array_equal(d.predict(x)["prob"], want)


def test_autotune_with_persistent_cache(gpu, tmp_path):
    """autotune times every tcgen05 tile configuration of each conv / linear (and dual GEMM)
    step on the plan's own buffers and keeps the fastest (dnn.cpp:214-290); the choices persist
    in a versioned TuneCache JSON, so a second compile measures nothing."""
    import json
    from paper_2003_10688_b200 import frontend, graph, models
    g = models.resnet(50, hw=64, classes=16, width=16)
    gi = graph.infer_shapes(g, 8)
    ins = _inputs(gi, 8, seed=7)
    path = str(tmp_path / "tune.json")
    frontend._TUNE_CACHE = frontend.TuneCache()
    m = frontend.optimize(g, _opts(fuse_epilogue=True, autotune=True, tune_budget=3, tune_cache_path=path))
    out = m.predict(ins)["prob"]
    assert m.tuner_runs > 0 and len(m.tuned) > 10
    assert O.oracle_err(out, O.run_graph(gi, ins)["prob"]) <= 1e-2
    d = json.load(open(path))
    assert d["version"] == frontend.TUNE_VERSION and len(d["entries"]) > 5
    assert any(e["choice"]["tile_n"] != 0 for e in d["entries"].values()) or all(
        len(e["candidates"]) > 1 for e in d["entries"].values())
    frontend._TUNE_CACHE = frontend.TuneCache()
    m2 = frontend.optimize(g, _opts(fuse_epilogue=True, autotune=True, tune_budget=3, tune_cache_path=path))
    out2 = m2.predict(ins)["prob"]
    assert m2.tuner_runs == 0 and m2.tune_cache_hits == len(m.tuned)
    assert np.array_equal(out, out2)


def test_export_and_run_bundle_bit_identical(gpu, tmp_path):
    from paper_2003_10688_b200 import frontend, graph
    g = _model(True)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=8)
    m = frontend.optimize(g, _opts(train=True, lr=0.05, fuse_epilogue=True))
    m.train_step(ins)
    x = {"x": ins["x"]}
    want = m.predict(x)["prob"]
    d = str(tmp_path / "bundle")
    man = m.export_bundle(d)
    with pytest.raises(FileExistsError):
        m.export_bundle(d)
    m.export_bundle(d, force=True)
    got = frontend.run_bundle(d, x)["prob"]
    assert man.endswith("manifest.json")
    assert np.array_equal(got, want)


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_fused_dgrad_relu_back_is_exact(gpu, dtype):
    """fusion.fuse_dgrad_relu_back: the stride-1 dgrads apply the ReluBack mask (inner ReLUs) or
    Add + ReluBack (block outputs) in their GEMM epilogue; the step (loss, every gradient) is
    bit-identical to the unfused plan's."""
    from paper_2003_10688_b200 import frontend, graph
    g = _model(True)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=9)
    a = frontend.optimize(g, _opts(dtype=dtype, train=True, lr=0.05))
    b = frontend.optimize(g, _opts(dtype=dtype, train=True, lr=0.05, fuse_relu_back=False))
    ops = [[a.graph.find_node(n).op for n in u.node_ids] for u in a.units if u.kind == "dnn"]
    fused = [o for o in ops if o[0] == "Conv2dBackX" and len(o) > 1]
    assert ["Conv2dBackX", "ReluBack"] in fused and ["Conv2dBackX", "Add", "ReluBack"] in fused
    assert len(a.units) == len(b.units) - len(fused)
    assert any(st.family == "conv_dgrad_fused_tcgen05" for st in a.steps)
    assert a.train_step(ins) == b.train_step(ins)
    ga, gb = a.gradients(), b.gradients()
    assert ga.keys() == gb.keys()
    for k in ga:
        assert np.array_equal(ga[k], gb[k]), k


def test_bn_stats_from_conv_epilogue(gpu):
    """bn_stats_from_conv: a training BatchNorm's batch statistics come out of the producing conv's
    GEMM epilogue (partial sums of (y - previous batch mean) per M tile and row quarter) instead of
    a pass over y. After several steps (the shift is then the previous step's mean), every linked
    BN unit's output matches the oracle BN of the plan's own conv output, and the loss follows the
    statistics-pass plan (bf16 rounding flips amplify through the network, hence the tolerance)."""
    import torch
    from paper_2003_10688_b200 import dfp, frontend, graph, models
    from tests.gpu_util import from_device
    g = models.resnet(50, hw=64, classes=16, width=16, train=True, seed=5)
    ins = _inputs(graph.infer_shapes(g, 8), 8, seed=10)
    a = frontend.optimize(g, _opts(train=True, lr=0.0, keep_all=True))
    b = frontend.optimize(g, _opts(train=True, lr=0.0, bn_stats_from_conv=False))
    pa = a._plan(True)
    assert pa.bn_stats_links > 20 and b._plan(True).bn_stats_links == 0
    assert any(st.family == "conv_fprop_bnstats_tcgen05" for st in pa.steps)
    for _ in range(3):
        la, lb = a.train_step(ins), b.train_step(ins)
    np.testing.assert_allclose(la, lb, rtol=2e-2)

    def get(nm):
        raw = pa.read_tensor(nm)
        f32 = dfp.is_f32_tensor(pa.graph, nm)
        t = torch.from_numpy(raw.view(np.float32).copy() if f32 else raw.view(np.int16).copy())
        return from_device(t if f32 else t.view(torch.bfloat16), pa.graph.meta_of(nm)).astype(np.float64)

    linked = {pa.steps[i].output for i in range(len(pa.steps)) if pa.steps[i].family == "conv_fprop_bnstats_tcgen05"}
    checked, bad = 0, []
    for u in pa.units:
        first = pa.graph.find_node(u.node_ids[0])
        if u.kind != "dfp" or first.op != "BatchNorm2d" or first.inputs[0] not in linked:
            continue
        local = {nm: get(nm) for nm in u.inputs}
        params = {k: np.asarray(v, np.float64) for k, v in pa.params.items()}
        for nid in u.node_ids:
            n = pa.graph.find_node(nid)
            local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
        err = O.oracle_err(get(u.output), local[u.output])
        checked += 1
        if err > 2e-2:
            bad.append((u.output, err))
    assert checked > 20 and not bad, bad
