"""Per-unit parity of every fused DFP kernel and tcgen05 provider against the oracle, on
oracle-supplied unit inputs (proj/tests/test_dfp.cpp:26-45, :223-270; test_autodiff.cpp:355-385).

Bars: f32 plans (fp32 DFP arithmetic) oracle_err <= 1e-5 for fused non-GEMM units — the
reference's own kernel bar; bit-exact for pure movement (Flatten, Concat); TF32 / bf16 GEMM
units and every bf16 unit <= 1e-2 against the oracle run on bf16-rounded unit inputs."""
import numpy as np
import pytest

from oracle import sol_oracle as O
from tests.gpu_util import quant, run_unit

pytestmark = pytest.mark.gpu

MOVEMENT = {"flatten", "flatten_back"}


def tf32(a):
    """TF32 operand rounding of the tcgen05 kind::tf32 path (low 13 mantissa bits dropped)."""
    a = np.ascontiguousarray(np.asarray(a, np.float32))
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


def _graphs():
    from paper_2003_10688_b200 import models
    return {
        "small_cnn": lambda tr: models.small_cnn(train=tr, hw=16),
        "resnet18": lambda tr: models.resnet(18, hw=32, classes=16, width=16, train=tr),
        "resnet50": lambda tr: models.resnet(50, hw=64, classes=16, width=16, train=tr),
        "densenet": lambda tr: models.densenet121(hw=32, classes=16, growth=8, blocks=(2, 3), init=16, train=tr),
        "mobilenet": lambda tr: models.mobilenet_v2(hw=32, classes=16, width_mult=0.5, train=tr),
    }


def _inputs(g, batch, seed=0):
    rng = np.random.default_rng(seed)
    ins = {}
    for gi in g.graph_inputs:
        if gi.name == "t":
            t = np.zeros(gi.meta.shape, np.float32)
            t[np.arange(batch), np.arange(batch) % gi.meta.shape[1]] = 1.0
            ins["t"] = t
        else:
            ins[gi.name] = rng.uniform(-1, 1, gi.meta.shape).astype(np.float32)
    return ins


def _compile(name, train, batch):
    from paper_2003_10688_b200 import autodiff, graph, partition, passes
    g = _graphs()[name](train)
    gi = graph.infer_shapes(g, batch)
    if train:
        gi = graph.infer_shapes(autodiff.build_training_graph(gi).graph, batch)
    gp = passes.run_pipeline(gi)
    return gp, partition.partition(gp)


def _check_units(gp, units, env, dtype, gpu, only_dfp=False):
    worst = {}
    for u in units:
        if only_dfp and u.kind != "dfp":
            continue
        # oracle output of this unit from (dtype-rounded) oracle inputs
        heavy = u.kind == "dnn"
        sub = {}
        for nm in u.inputs:
            sub[nm] = quant(env[nm], dtype) if dtype == 1 else env[nm]
            if heavy and dtype == 0:
                sub[nm] = tf32(sub[nm])
        params = {k: np.asarray(v, np.float64) for k, v in gp.params.items()}
        if heavy:
            # the tensor cores read W in the operand precision
            for pn in u.params:
                if gp.params[pn].ndim >= 2:
                    params[pn] = (tf32 if dtype == 0 else (lambda a: quant(a, 1)))(gp.params[pn]).astype(np.float64)
        local = dict(sub)
        for nid in u.node_ids:
            n = gp.find_node(nid)
            local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
        want = np.asarray(local[u.output], np.float32)
        fam, got = run_unit(gp, u, env, dtype, gpu)
        if fam in ("bias_grad", "bn_back_beta", "bn_back_gamma"):
            # channel sums with heavy cancellation (a conv bias feeding a training BatchNorm has an
            # analytically ~0 gradient): measure the error against the sum of |terms| per channel
            d = np.asarray(sub[u.inputs[0]], np.float64)
            terms = np.abs(d)
            if fam == "bn_back_gamma":
                x = np.asarray(sub[u.inputs[1]], np.float64)
                mu, var = O.batch_stats(x)
                terms = np.abs(d * (x - O._bc(mu, x)) / np.sqrt(O._bc(var, x) + 1e-5))
            l1 = terms.sum(axis=(0, 2, 3) if terms.ndim == 4 else (0,))
            bar = 1e-2 if dtype == 1 else 1e-6
            assert np.max(np.abs(got - want)) <= bar * np.max(l1), (fam, u.output)
            continue
        err = O.oracle_err(got, want)
        if fam in MOVEMENT:
            assert np.array_equal(got.astype(np.float32), want.astype(np.float32)), (fam, u.output)
        bar = 1e-2 if (dtype == 1 or heavy) else 1e-5
        if fam == "bn_back_x" and dtype == 0:
            # dx = g*rstd*(dy - mean(dy) - xhat*mean(dy*xhat)) cancels against dy when the batch is
            # small (m = 16 here); f32 arithmetic then carries ~|dy|/|dx| * 6e-8 relative error
            bar = 5e-5
        assert err <= bar, (fam, u.output, u.node_ids, err)
        worst[fam] = max(worst.get(fam, 0.0), err)
    return worst


@pytest.mark.parametrize("name", ["small_cnn", "resnet18", "resnet50", "densenet", "mobilenet"])
@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_inference_units(gpu, name, dtype):
    batch = 3
    gp, units = _compile(name, False, batch)
    env = O.run_graph(gp, _inputs(gp, batch))
    _check_units(gp, units, env, dtype, gpu)


@pytest.mark.parametrize("name", ["small_cnn", "resnet18", "resnet50"])
@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_training_units(gpu, name, dtype):
    batch = 4
    gp, units = _compile(name, True, batch)
    env = O.run_graph(gp, _inputs(gp, batch))
    _check_units(gp, units, env, dtype, gpu)


@pytest.mark.parametrize("hw,k,s,p,bias", [(64, 7, 2, 3, False), (37, 7, 2, 3, True), (30, 3, 1, 1, True),
                                            (33, 3, 2, 1, False)])
def test_stem_conv(gpu, hw, k, s, p, bias):
    """Few-channel stem conv (3 -> 64, stem.cu halo-tile kernel) vs the oracle on bf16 operands;
    ragged sizes exercise partial output tiles and the out-of-bounds halo fill."""
    from paper_2003_10688_b200 import graph, partition
    b = graph.GraphBuilder(21)
    b.input("x", graph.meta_nchw(0, 3, hw, hw))
    c = b.conv("stem", "x", 3, 64, k, s, p, bias=bias)
    batch = 3
    g = graph.infer_shapes(b.done([c]), batch)
    units = partition.partition(g)
    x = np.random.default_rng(4).uniform(-1, 1, (batch, 3, hw, hw)).astype(np.float32)
    fam, got = run_unit(g, units[0], {"x": x}, 1, gpu)
    assert fam == "conv_stem_tcgen05"
    params = {k2: np.asarray(quant(v, 1) if v.ndim >= 2 else v, np.float64) for k2, v in g.params.items()}
    want = O.eval_node(g.find_node("stem"), [quant(x, 1).astype(np.float64)], params)
    err = O.oracle_err(got, want)
    assert got.shape == want.shape and err <= 1e-2, err


@pytest.mark.parametrize("hw", [64, 37])
def test_stem_wgrad(gpu, hw):
    """Stem weight gradient (stem.cu WG mode: halo im2col tiles as the MN-major operand, per-CTA
    TMEM accumulation, f32 partial reduction) vs the oracle's Conv2dBackW on bf16 operands."""
    from paper_2003_10688_b200 import autodiff, graph, partition, passes
    b = graph.GraphBuilder(23)
    b.input("x", graph.meta_nchw(0, 3, hw, hw))
    c = b.conv("stem", "x", 3, 64, 7, 2, 3, bias=False)
    p = b.node("gap", "GlobalAvgPool", [c], graph.Attrs())
    f = b.linear("fc", p, 64, 8)
    prob = b.softmax("prob", f)
    b.input("t", graph.meta_nc(0, 8))
    batch = 3
    g = graph.infer_shapes(b.done([b.ce("loss", prob, "t")]), batch)
    tg = graph.infer_shapes(autodiff.build_training_graph(g).graph, batch)
    gp = passes.run_pipeline(tg)
    units = partition.partition(gp)
    ins = _inputs(gp, batch, seed=6)
    env = O.run_graph(gp, ins)
    u = next(u for u in units if gp.find_node(u.node_ids[0]).op == "Conv2dBackW")
    local = {nm: quant(env[nm], 1).astype(np.float64) for nm in u.inputs}
    params = {k: np.asarray(v, np.float64) for k, v in gp.params.items()}
    for nid in u.node_ids:
        n = gp.find_node(nid)
        local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
    fam, got = run_unit(gp, u, env, 1, gpu)
    assert fam == "conv_stem_wgrad_tcgen05"
    err = O.oracle_err(got, local[u.output])
    assert err <= 1e-2, err


@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_maxpool_back_band_stem_scale(gpu, monkeypatch, dtype):
    """The ResNet stem's MaxPool2dBack (+ReluBack) unit at 224x224 (112x112 -> 56x56, 3x3/2/1):
    the one-pass band kernel matches the oracle and is bit-identical to the two-pass
    argmax + gather path (SOL_NO_POOLBACK_BAND=1). Inputs on a coarse grid so windows hold ties
    (first-max routing, reference.cpp:294-327) and ReLU zeros (min_init routes nothing)."""
    from paper_2003_10688_b200 import models
    from paper_2003_10688_b200 import autodiff, graph, partition, passes
    batch = 2
    g = models.resnet(18, hw=224, classes=16, width=16, train=True)
    gi = graph.infer_shapes(g, batch)
    gi = graph.infer_shapes(autodiff.build_training_graph(gi).graph, batch)
    gp = passes.run_pipeline(gi)
    units = [u for u in partition.partition(gp)
             if any(gp.find_node(nid).op == "MaxPool2dBack" for nid in u.node_ids)]
    assert len(units) == 1
    u = units[0]
    rng = np.random.default_rng(5)
    env = {}
    for nm in u.inputs:
        shape = gp.meta_of(nm).shape
        env[nm] = (rng.integers(-3, 5, shape) / 4.0).astype(np.float32)
    _check_units(gp, [u], env, dtype, gpu)
    fam, band = run_unit(gp, u, env, dtype, gpu)
    assert fam == "dfp_maxpool_back"
    monkeypatch.setenv("SOL_NO_POOLBACK_BAND", "1")
    _, two_pass = run_unit(gp, u, env, dtype, gpu)
    assert np.array_equal(band, two_pass)


@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_maxpool_bulk_stem_scale(gpu, monkeypatch, dtype):
    """The ResNet stem's inference BatchNorm + MaxPool unit at 224x224 (112x112 -> 56x56, 3x3/2/1)
    on the bulk band kernel: matches the oracle, and is bit-identical to the per-tap row kernel
    (SOL_POOL_BAND=0). The bf16 band kernel reduces raw taps with packed max / min and maps the
    BatchNorm once (monotone map): gammas of both signs and a zero, inputs on a coarse grid so
    windows hold ties, so both the max and the min branch are exercised."""
    from paper_2003_10688_b200 import models
    from paper_2003_10688_b200 import graph, partition, passes
    batch = 2
    g = models.resnet(18, hw=224, classes=16, width=16)
    gp = passes.run_pipeline(graph.infer_shapes(g, batch))
    units = [u for u in partition.partition(gp)
             if any(gp.find_node(nid).op == "MaxPool2d" for nid in u.node_ids)]
    assert len(units) == 1
    u = units[0]
    rng = np.random.default_rng(11)
    for pn in u.params:
        c = gp.params[pn].shape[0]
        if pn.endswith("gamma"):
            gam = rng.uniform(0.25, 2.0, c) * np.where(rng.random(c) < 0.5, -1.0, 1.0)
            gam[0] = 0.0
            gp.params[pn] = gam.astype(np.float32)
        elif pn.endswith("beta") or pn.endswith("running_mean"):
            gp.params[pn] = rng.uniform(-1, 1, c).astype(np.float32)
        elif pn.endswith("running_var"):
            gp.params[pn] = rng.uniform(0.5, 2.0, c).astype(np.float32)
    env = {nm: (rng.integers(-4, 5, gp.meta_of(nm).shape) / 4.0).astype(np.float32) for nm in u.inputs}
    _check_units(gp, [u], env, dtype, gpu)
    fam, bulk = run_unit(gp, u, env, dtype, gpu)
    assert fam == "dfp_maxpool"
    monkeypatch.setenv("SOL_POOL_BAND", "0")
    _, rowk = run_unit(gp, u, env, dtype, gpu)
    assert np.array_equal(bulk, rowk)


@pytest.mark.parametrize("dtype", [0, 1], ids=["f32", "bf16"])
def test_gap_back_relu_back_mask_kernel(gpu, monkeypatch, dtype):
    """ResNet-50's last training unit, GlobalAvgPoolBack + ReluBack (dx = relu_out > 0 ? g[n, c] /
    (H*W) : 0), on the mask kernel with an [N, C] broadcast source: matches the oracle and is
    bit-identical to the generic DFP interpreter (SOL_NO_MASK_KERNEL=1)."""
    from paper_2003_10688_b200 import models
    from paper_2003_10688_b200 import autodiff, graph, partition, passes
    batch = 4
    g = models.resnet(50, hw=64, classes=16, width=16, train=True)
    gi = graph.infer_shapes(g, batch)
    gi = graph.infer_shapes(autodiff.build_training_graph(gi).graph, batch)
    gp = passes.run_pipeline(gi)
    units = [u for u in partition.partition(gp)
             if any(gp.find_node(nid).op == "GlobalAvgPoolBack" for nid in u.node_ids)]
    assert len(units) == 1
    u = units[0]
    rng = np.random.default_rng(3)
    env = {nm: rng.uniform(-1, 1, gp.meta_of(nm).shape).astype(np.float32) for nm in u.inputs}
    _check_units(gp, [u], env, dtype, gpu)
    fam, fast = run_unit(gp, u, env, dtype, gpu)
    monkeypatch.setenv("SOL_NO_MASK_KERNEL", "1")
    _, generic = run_unit(gp, u, env, dtype, gpu)
    assert np.array_equal(fast, generic)
