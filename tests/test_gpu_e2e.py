"""End-to-end parity of the network API (optimize -> predict / train_step) against the oracle.

Bars (north star): bf16/TF32 end-to-end max relative error <= 1e-2 (oracle_err metric) on the
outputs and 100% top-1 agreement where the oracle's top-1 margin exceeds that band."""
import numpy as np
import pytest

from oracle import sol_oracle as O
from tests.test_gpu_units import _graphs, _inputs

pytestmark = pytest.mark.gpu


def _top1_ok(got, want, tol=1e-2):
    srt = np.sort(want, axis=1)
    margin = (srt[:, -1] - srt[:, -2]) / np.maximum(np.abs(srt[:, -1]), 1e-12)
    clear = margin > 4 * tol
    return np.all(np.argmax(got, 1)[clear] == np.argmax(want, 1)[clear]), int(clear.sum())


@pytest.mark.parametrize("name", ["small_cnn", "resnet18", "resnet50", "densenet", "mobilenet"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("fuse", [False, True], ids=["units", "fused"])
def test_predict(gpu, name, dtype, fuse):
    from paper_2003_10688_b200 import frontend, graph
    batch = 4
    g = _graphs()[name](False)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype=dtype, fuse_epilogue=fuse))
    ins = _inputs(graph.infer_shapes(g, batch), batch, seed=5)
    out = m.predict(ins)
    env = O.run_graph(graph.infer_shapes(g, batch), ins)
    got, want = out["prob"], env["prob"]
    err = O.oracle_err(got, want)
    print(f"e2e {name} {dtype}: oracle_err(prob) = {err:.3e}")
    assert err <= 1e-2
    ok, n = _top1_ok(got, want)
    assert ok, n
    # graph replay gives the identical answer
    out2 = m.predict(ins)
    assert np.array_equal(out2["prob"], got)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("name,hw", [("small_cnn", 32), ("resnet18", 64), ("resnet50", 64)])
def test_train_step(gpu, name, hw, dtype):
    """Native training step: loss within 2% of the oracle, every parameter gradient with a
    cosine similarity >= 0.95 to the oracle's for every conv/linear weight (bf16 activations
    compound rounding through the backward chain, so elementwise relative error is not a meaningful
    bar here; per-unit parity in test_gpu_units and the composition check below hold the strict
    bars; BatchNorm affine gradients are sums with heavy cancellation at random init and are
    reported, not asserted), SGD applied on the device, loss decreasing."""
    from paper_2003_10688_b200 import autodiff, frontend, graph, models
    batch = 16
    if name == "small_cnn":
        g = models.small_cnn(train=True, hw=hw)
    else:
        g = models.resnet(18 if name == "resnet18" else 50, hw=hw, classes=16, width=16, train=True)
    lr = 0.005
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype=dtype, train=True, lr=lr))
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=9)
    loss = m.train_step(ins)
    grads = m.gradients()
    tg = autodiff.build_training_graph(gi)
    env = O.run_graph(graph.infer_shapes(tg.graph, batch), ins)
    ref_loss = float(env[tg.loss])
    assert abs(loss - ref_loss) <= 2e-2 * abs(ref_loss), (loss, ref_loss)
    worst = []
    for p, gname in tg.param_grads:
        want = np.asarray(env[gname], np.float64).ravel()
        got = grads[p].astype(np.float64).ravel()
        if np.linalg.norm(want) < 1e-4 * np.sqrt(want.size):
            continue  # gradient is cancellation noise (e.g. conv bias before BatchNorm)
        cos = float(got @ want / (np.linalg.norm(got) * np.linalg.norm(want) + 1e-30))
        worst.append((cos, p))
    worst.sort()
    weights = [w for w in worst if g.params[w[1]].ndim >= 2]
    # conditioning floor: the oracle's own gradient cosine when its weights carry the rounding of
    # the tensor-core path (TF32 ~5e-4 relative; bf16 4e-3: bf16 rounds the weights AND every
    # stored activation, 2^-9 each), worst of two perturbations. Deep random-init BatchNorm nets are
    # ill-conditioned (ResNet-50 here: ~0.7 / ~0.3), so the bar is relative to this floor.
    rel = 5e-4 if dtype == "f32" else 4e-3
    gp = graph.infer_shapes(tg.graph, batch)
    floor = 1.0
    for seed in (1, 2):
        rng = np.random.default_rng(seed)
        gp.params = {k: (v * (1 + rel * rng.standard_normal(v.shape))).astype(np.float32)
                     for k, v in g.params.items()}
        env2 = O.run_graph(gp, ins)
        floor = min(floor, min(float(np.dot(env[gn].ravel(), env2[gn].ravel()) /
                                     (np.linalg.norm(env[gn]) * np.linalg.norm(env2[gn]) + 1e-30))
                               for p, gn in tg.param_grads if g.params[p].ndim >= 2))
    print(f"{name} {dtype}: min grad cosine conv/linear {weights[0][0]:.4f} "
          f"(oracle self-consistency under operand rounding {floor:.4f}), all params {worst[0][0]:.4f}")
    # measured (B200): the plan is never below the floor (small CNN 0.994 vs 0.993, ResNet-18 bf16
    # 0.923 vs 0.908, ResNet-50 f32 0.819 vs 0.694), so the bar sits at 90% of it (0.95 cap)
    assert weights[0][0] >= min(0.95, 0.9 * floor), weights[:5]
    new = m.host_params()
    for p, _ in tg.param_grads[:8]:
        np.testing.assert_allclose(new[p], g.params[p] - np.float32(lr) * grads[p], rtol=1e-5, atol=1e-6)
    losses = [m.train_step(ins) for _ in range(5)]
    assert losses[-1] < loss, losses


def _bf16(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("name", ["small_cnn", "resnet18", "resnet50"])
def test_plan_composition(gpu, name):
    """Every unit of a composed training plan, re-evaluated by the oracle on the plan's own input
    buffers (weights rounded to bf16 for the tensor-core units), matches the plan's output buffer:
    isolates wiring / arena-placement errors from precision."""
    import torch
    from paper_2003_10688_b200 import dfp, frontend, graph, models
    from tests.gpu_util import from_device
    batch = 8
    g = models.small_cnn(train=True, hw=32) if name == "small_cnn" else \
        models.resnet(18 if name == "resnet18" else 50, hw=64, classes=16, width=16, train=True)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=True, lr=0.0,
                                                      keep_all=True))
    m.train_step(_inputs(graph.infer_shapes(g, batch), batch, seed=3))

    def get(nm):
        meta = m.graph.meta_of(nm)
        raw = m.read_tensor(nm)
        f32 = dfp.is_f32_tensor(m.graph, nm)
        t = torch.from_numpy(raw.view(np.float32).copy() if f32 else raw.view(np.int16).copy())
        return from_device(t if f32 else t.view(torch.bfloat16), meta).astype(np.float64)

    bad = []
    for u in m.units:
        params = {k: np.asarray(_bf16(v) if (u.kind == "dnn" and v.ndim >= 2) else v, np.float64)
                  for k, v in m.params.items()}
        local = {nm: get(nm) for nm in u.inputs}
        for nid in u.node_ids:
            n = m.graph.find_node(nid)
            local[nid] = O.eval_node(n, [local[i] for i in n.inputs], params)
        got = get(u.output)
        err = O.oracle_err(got, local[u.output])
        if len(u.node_ids) == 3 and m.graph.find_node(u.node_ids[0]).op == "Conv2dBackX":
            # fused dgrad + Add + ReluBack (fusion.fuse_dgrad_relu_back; bit-identical to the unfused
            # plan): the sum of two gradients cancels, so one bf16 ulp of the rounded dgrad is
            # measured against the operands' magnitude, not the (possibly tiny) sum's
            add = m.graph.find_node(u.node_ids[1])
            mag = np.abs(local[add.inputs[0]]) + np.abs(local[add.inputs[1]])
            den = np.maximum(mag, max(0.01 * float(mag.max()), 1e-12))
            err = float(np.max(np.abs(got - local[u.output]) / den))
        if not np.all(np.isfinite(got)) or err > 2e-2:
            bad.append((u.output, err))
    assert not bad, bad


def test_pipelined_staging_matches_predict(gpu):
    """stage_inputs() (copy-stream H2D of the next batch overlapping the current run) gives the
    same answers as predict(), batch after batch."""
    from paper_2003_10688_b200 import frontend, graph, models
    batch = 4
    g = models.resnet(18, hw=32, classes=16, width=16)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True))
    gi = graph.infer_shapes(g, batch)
    batches = [_inputs(gi, batch, seed=s) for s in (11, 12, 13)]
    want = [m.predict(b)["prob"] for b in batches]
    got = []
    for b in batches:
        m.stage_inputs(b)
        m.run()
        got.append(m.fetch_outputs(["prob"])["prob"])
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    # serving order: the next batch is staged (pinned slot refilled on the host) while the current
    # run is still in flight, BEFORE its outputs are fetched; each answer must still be its own
    # batch's (the pinned slots alternate and are refilled only after their copy completed)
    batches = [_inputs(gi, batch, seed=s) for s in range(20, 27)]
    want = [m.predict(b)["prob"] for b in batches]
    m.stage_inputs(batches[0])
    for i in range(len(batches)):
        m.run()
        if i + 1 < len(batches):
            m.stage_inputs(batches[i + 1])
        assert np.array_equal(m.fetch_outputs(["prob"])["prob"], want[i]), i
    # zero-copy slots: fill input_buffers() in place, then stage without an argument
    for i in (3, 4):
        for name, v in m.input_buffers().items():
            v[...] = batches[i][name]
        m.stage_inputs()
        m.run()
        assert np.array_equal(m.fetch_outputs(["prob"])["prob"], want[i]), i


@pytest.mark.parametrize("stride,conv_bias", [(1, False), (2, False), (2, True)])
def test_bottleneck_dual_gemm(gpu, stride, conv_bias):
    """Bottleneck tail + downsample fused into one dual GEMM (fusion.fuse_bottleneck_tails): both
    BN scales folded into bf16 weights, stride-2 downsample read by TMA im2col; predict() matches
    the oracle within the bf16 bar and the unfused plan's answers."""
    from paper_2003_10688_b200 import frontend, graph
    from paper_2003_10688_b200.models import _bottleneck, _head
    b = graph.GraphBuilder(31)
    b.input("x", graph.meta_nchw(0, 64, 16, 16))
    y, cout = _bottleneck(b, "x", 64, 64, stride, "blk")
    if conv_bias:
        for k in ("blk.conv3.b", "blk.down.b"):
            b.g.params[k] = np.random.default_rng(2).uniform(-0.2, 0.2, cout).astype(np.float32)
        for nid in ("blk.conv3", "blk.down"):
            n = next(n for n in b.g.nodes if n.id == nid)
            n.attrs.has_bias = True
            n.params = [nid + ".W", nid + ".b"]
    y = b.conv("tail", y, cout, 64, 1, 1, 0)  # a heavy consumer keeps the block's ReLU unit closed
    p = b.gap("gap", y)
    g = _head(b, p, 64, 10, False)
    batch = 4
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=7)
    fused = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True))
    assert any(len(u.node_ids) >= 5 for u in fused.units), "dual GEMM unit not formed"
    plain = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16"))
    got, ref = fused.predict(ins)["prob"], plain.predict(ins)["prob"]
    want = O.run_graph(gi, ins)["prob"]
    assert O.oracle_err(got, want) <= 1e-2
    assert O.oracle_err(got, ref) <= 1e-2


@pytest.mark.parametrize("bucket_mb", ["25", "0.02"])
def test_nccl_allreduce_plumbing_single_rank(gpu, monkeypatch, bucket_mb):
    """The data-parallel training plan (NCCL all-reduce of every gradient in ~bucket_mb buckets,
    ncclAvg, each bucket issued on the comm stream right after the unit completing its last
    gradient so it overlaps the rest of the backward pass, joined before SGD; all inside the
    captured CUDA graph) run with one replica: must reproduce the plain plan bit for bit.
    (Multi-replica runs need one process per GPU; this box has one GPU.)"""
    from paper_2003_10688_b200 import frontend, graph, models
    monkeypatch.setenv("SOL_AR_BUCKET_MB", bucket_mb)
    batch = 8
    g = models.resnet(18, hw=32, classes=16, width=16, train=True)
    ins = _inputs(graph.infer_shapes(g, batch), batch, seed=4)
    res = []
    for force in (False, True):
        m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", train=True, lr=0.01,
                                                          nccl_allreduce=force))
        if force:
            ar = [i for i, st in enumerate(m.steps) if st.kind == "allreduce"]
            assert len(ar) == len(m.param_grads)
            if bucket_mb != "25":  # small buckets interleave with the backward units
                assert m.ar_buckets > 1 and ar[0] < min(i for i, st in enumerate(m.steps) if st.kind == "sgd") - 10
        losses = [m.train_step(ins) for _ in range(3)]
        res.append((losses, m.host_params()))
    assert res[0][0] == res[1][0]
    for k in res[0][1]:
        assert np.array_equal(res[0][1][k], res[1][1][k]), k


def test_direct_nchw_stem_input(gpu, monkeypatch):
    """A bf16 inference plan whose stem is the graph input's only consumer skips the reorder pass:
    the stem's halo TMA reads the canonical NCHW f32 input (ragged 60x60 images: partial tiles)."""
    from paper_2003_10688_b200 import frontend, graph, models
    batch = 3
    g = models.resnet(18, hw=60, classes=16, width=64)
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=12)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True))
    assert not any(st.kind == "reorder" and st.output == "x" for st in m.steps)
    assert any(st.family.startswith("conv_stem") for st in m.steps)
    got = m.predict(ins)["prob"]
    monkeypatch.setenv("SOL_NO_DIRECT_STEM", "1")
    ref = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True)).predict(ins)["prob"]
    want = O.run_graph(gi, ins)["prob"]
    assert O.oracle_err(got, want) <= 1e-2
    assert O.oracle_err(got, ref) <= 1e-2


@pytest.mark.parametrize("hw", [60, 224])
def test_stem_conv_pool_fusion(gpu, monkeypatch, hw):
    """Opt-in plan fusion (SOL_STEM_POOL=1): stem conv + BN + 3x3/2 max pool in one stem_row.cu
    launch that pools its own output rows in shared memory (bands of pooled rows, one recomputed conv
    row per band). The fused kernel applies the BN to the f32 accumulator before the one bf16
    rounding (the unfused plan rounds the raw conv output first), so the two plans agree to bf16
    rounding drift, and both match the oracle within the bf16 tolerance."""
    from paper_2003_10688_b200 import frontend, graph, models
    batch = 2
    g = models.resnet(18, hw=hw, classes=16, width=64)
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=21)
    opts = frontend.OptimizeOptions(batch=batch, dtype="bf16", fuse_epilogue=True)
    ref = frontend.optimize(g, opts)
    monkeypatch.setenv("SOL_STEM_POOL", "1")
    m = frontend.optimize(g, opts)
    fused = [st for st in m.steps if st.family.startswith("conv_stem")]
    assert len(fused) == 1 and not any(st.family == "dfp_maxpool" for st in m.steps)
    got = m.predict(ins)["prob"]
    want = ref.predict(ins)["prob"]
    assert O.oracle_err(got, want) <= 1e-2
    if hw <= 64:  # the f64 oracle at 224x224 takes minutes; the unfused plan is oracle-checked elsewhere
        assert O.oracle_err(got, O.run_graph(gi, ins)["prob"]) <= 1e-2


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_train_step_updates_bn_running_stats(gpu, dtype):
    """Native training applies update_bn_running_stats (autodiff.cpp:356-384) on the device: after
    one step every running_mean / running_var equals the oracle's update computed from the plan's
    own BatchNorm input tensors (f64 statistics, momentum 0.1, unbiased variance); a second step
    applies it again; inference after training uses the updated statistics."""
    import torch
    from paper_2003_10688_b200 import dfp, frontend, graph, models
    from tests.gpu_util import from_device
    batch = 8
    g = models.resnet(18, hw=32, classes=16, width=16, train=True)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=batch, dtype=dtype, train=True, lr=0.0, keep_all=True))
    gi = graph.infer_shapes(g, batch)
    ins = _inputs(gi, batch, seed=19)

    def get(nm):
        raw = m.read_tensor(nm)
        f32 = dtype == "f32" or dfp.is_f32_tensor(m.graph, nm)
        t = torch.from_numpy(raw.view(np.float32).copy() if f32 else raw.view(np.int16).copy())
        return from_device(t if f32 else t.view(torch.bfloat16), m.graph.meta_of(nm)).astype(np.float64)

    params = {k: v.copy() for k, v in g.params.items()}
    for step in range(2):
        m.train_step(ins)
        env = {n.inputs[0]: get(n.inputs[0]) for n in m.graph.nodes if n.op == "BatchNorm2d" and n.attrs.training}
        params = O.update_bn_running_stats(m.graph, params, env)
        got = m.host_params()
        names = [k for k in params if k.endswith(("running_mean", "running_var"))]
        assert len(names) == 2 * sum(1 for n in m.graph.nodes if n.op == "BatchNorm2d")
        for k in names:
            np.testing.assert_allclose(got[k], params[k], rtol=2e-5, atol=1e-6, err_msg=f"step {step} {k}")
        for k in names:
            params[k] = got[k]  # the next step starts from the device's values
