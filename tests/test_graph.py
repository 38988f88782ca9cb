"""Host-side graph logic against the reference (CPU only):
 * partition parity: the B200 planner produces exactly the reference's execution units
   (dfp_lower.cpp:70-165) after the same pass pipeline (passes.cpp), for inference and training
   graphs (fixtures tests/golden/partition_*.json written by scripts/make_golden.py from the
   reference library itself);
 * autodiff parity: the same training graph node sequence and parameter -> gradient map
   (autodiff.cpp);
 * the model JSON / SOLW weight formats round-trip (model_io.cpp, weights_io.cpp);
 * the conv-epilogue fusion pass only merges what it may."""
import json
import os

import numpy as np
import pytest

from paper_2003_10688_b200 import autodiff, graph, models, partition, passes
from paper_2003_10688_b200.graph import MalformedModelError

GOLD = os.path.join(os.path.dirname(__file__), "golden")

CASES = {
    "resnet50": (lambda: models.resnet(50), False),
    "resnet50_train": (lambda: models.resnet(50, train=True), True),
    "resnet18": (lambda: models.resnet(18), False),
    "small_cnn": (lambda: models.small_cnn(), False),
    "small_cnn_train": (lambda: models.small_cnn(train=True), True),
}


def _compiled(build, training, batch=2):
    g = build()
    gi = graph.infer_shapes(g, batch)
    grads = []
    if training:
        tg = autodiff.build_training_graph(gi)
        gi = graph.infer_shapes(tg.graph, batch)
        grads = [list(p) for p in tg.param_grads]
    cg = passes.run_pipeline(gi)
    return g, cg, partition.partition(cg), grads


@pytest.mark.parametrize("name", sorted(CASES))
def test_partition_matches_reference(name):
    with open(os.path.join(GOLD, f"partition_{name}.json")) as f:
        gold = json.load(f)
    _, cg, units, grads = _compiled(*CASES[name])
    assert [n.id for n in cg.nodes] == [n["id"] for n in gold["graph"]["nodes"]]
    assert [n.op for n in cg.nodes] == [n["op"] for n in gold["graph"]["nodes"]]
    assert len(units) == len(gold["units"])
    for u, w in zip(units, gold["units"]):
        assert u.kind == w["kind"], (u.output, w["output"])
        assert u.node_ids == w["node_ids"]
        assert u.output == w["output"]
        assert u.inputs == w["inputs"]
        assert u.params == w["params"]
    assert sorted(map(tuple, grads)) == sorted(map(tuple, gold["param_grads"]))


def test_fuse_relu_pool_sets_min_init():
    """passes.cpp fuse_relu_pool: ReLU -> MaxPool collapses into MaxPool(min_init=0)."""
    g = models.small_cnn()
    gi = graph.infer_shapes(g, 2)
    cg = passes.run_pipeline(gi)
    pools = [n for n in cg.nodes if n.op == "MaxPool2d"]
    assert pools and all(p.attrs.min_init == 0.0 for p in pools)
    assert len(cg.nodes) < len(gi.nodes)


@pytest.mark.parametrize("build", [lambda: models.small_cnn(),
                                   lambda: models.resnet(18, hw=32, classes=10, width=8),
                                   lambda: models.mobilenet_v2(hw=32, classes=10, width_mult=0.5),
                                   lambda: models.densenet121(hw=32, classes=8, growth=8, blocks=(2, 2), init=16)])
def test_model_json_and_weights_round_trip(build):
    g = build()
    text = graph.model_to_json(g)
    blob = graph.weights_to_bytes(g.params)
    g2 = graph.model_from_json(text, blob)
    assert graph.model_to_json(g2) == text
    assert sorted(g2.params) == sorted(g.params)
    for k, v in g.params.items():
        assert g2.params[k].dtype == np.float32 and np.array_equal(g2.params[k], v)


def test_weights_format_rejects_corruption():
    g = models.small_cnn()
    blob = bytearray(graph.weights_to_bytes(g.params))
    with pytest.raises(Exception):
        graph.weights_from_bytes(bytes(blob[:-3]))
    blob[0:4] = b"XXXX"
    with pytest.raises(Exception):
        graph.weights_from_bytes(bytes(blob))


def test_malformed_model_rejected():
    g = models.small_cnn()
    d = json.loads(graph.model_to_json(g))
    d["nodes"][1]["inputs"] = ["does_not_exist"]
    with pytest.raises(MalformedModelError):
        graph.infer_shapes(graph.model_from_json(json.dumps(d), graph.weights_to_bytes(g.params)), 2)


def test_training_graph_structure():
    """Every trainable parameter gets exactly one gradient node; softmax + CE backward is fused
    into one SoftmaxCeBack (autodiff.cpp); BN runs in training mode."""
    g = models.resnet(18, hw=32, classes=10, width=8, train=True)
    gi = graph.infer_shapes(g, 2)
    tg = autodiff.build_training_graph(gi)
    trainable = {p for p in g.params if not p.endswith(("running_mean", "running_var"))}
    assert {p for p, _ in tg.param_grads} == trainable
    ops = [n.op for n in tg.graph.nodes]
    assert ops.count("SoftmaxCeBack") == 1 and "SoftmaxBack" not in ops
    assert all(n.attrs.training for n in tg.graph.nodes if n.op == "BatchNorm2d")


def test_conv_epilogue_fusion():
    """Conv -> BN(inference) [-> Add] [-> ReLU] units merge into one fused heavy unit; a conv whose
    output has another consumer is left alone; ResNet-50 goes 108 -> 57 units."""
    from paper_2003_10688_b200.fusion import fuse_conv_epilogues
    g = models.resnet(50)
    cg = passes.run_pipeline(graph.infer_shapes(g, 2))
    units = partition.partition(cg)
    fused = fuse_conv_epilogues(cg, units)
    assert len(units) == 108 and len(fused) == 57
    # every node is still computed exactly once, in an order that respects dependencies
    seen = set(i.name for i in cg.graph_inputs)
    flat = []
    for u in fused:
        for nid in u.node_ids:
            n = cg.find_node(nid)
            assert all(i in seen or i in u.node_ids for i in n.inputs), nid
            flat.append(nid)
        seen.update(u.node_ids)
    assert sorted(flat) == sorted(n.id for n in cg.nodes)
    for u in fused:
        if u.kind == "dnn" and len(u.node_ids) > 1:
            ops = [cg.find_node(n).op for n in u.node_ids]
            assert ops[0] in ("Conv2d", "Linear") and ops[1] == "BatchNorm2d"
            assert set(ops[2:]) <= {"Add", "ReLU", "ReLU6"}


def test_tune_cache_roundtrip_and_version(tmp_path):
    """dnn::TuneCache semantics (dnn.hpp:104-121): keyed by hyperparameters, persisted as
    versioned JSON; a missing file is an empty cache, another version is ignored."""
    import json
    from paper_2003_10688_b200 import frontend, graph, models, partition
    g = graph.infer_shapes(models.resnet(18, hw=32, classes=10, width=8), 2)
    units = [u for u in partition.partition(g) if u.kind == "dnn"]
    keys = {frontend.TuneCache.key(g, u, 1, "B200") for u in units}
    assert len(keys) < len(units)  # repeated layer shapes share one key (no node ids in it)
    c = frontend.TuneCache()
    c.load(str(tmp_path / "missing.json"))
    assert c.size() == 0
    for i, k in enumerate(sorted(keys)):
        c.put(k, {"choice": {"tile_n": 128}, "micros": float(i)})
    p = str(tmp_path / "t.json")
    c.save(p)
    d = frontend.TuneCache()
    d.load(p)
    assert d.size() == len(keys) and d.find(sorted(keys)[1])["micros"] == 1.0
    j = json.load(open(p))
    j["version"] = 99
    json.dump(j, open(p, "w"))
    e = frontend.TuneCache()
    e.load(p)
    assert e.size() == 0


def test_options_fingerprint_tracks_plan_fields(monkeypatch):
    from paper_2003_10688_b200 import frontend
    monkeypatch.delenv("SOL_NO_DUAL", raising=False)
    a = frontend.OptimizeOptions(batch=4)
    fp0 = a.fingerprint()
    assert fp0 == frontend.OptimizeOptions(batch=4).fingerprint()
    assert fp0 != frontend.OptimizeOptions(batch=8).fingerprint()
    assert fp0 == frontend.OptimizeOptions(batch=4, tune_cache_path="/x").fingerprint()
    monkeypatch.setenv("SOL_NO_DUAL", "1")  # plan-changing switches are part of the key
    assert fp0 != a.fingerprint() and "SOL_NO_DUAL" in a.fingerprint()


def test_relu_mask_from_output_is_exact_and_fuses():
    """The training rewrite ReluBack(d, x) -> ReluBack(d, relu(x)) (and ReLU6Back) leaves every
    oracle gradient bit-identical and lets partition() fuse BN [+ Add] + ReLU (fewer units)."""
    import numpy as np
    from oracle import sol_oracle as O
    from paper_2003_10688_b200 import autodiff, graph, models, partition, passes
    for g in (models.resnet(18, hw=16, classes=10, width=8, train=True),
              models.mobilenet_v2(hw=32, classes=10, width_mult=0.5, train=True)):
        hw = g.graph_inputs[0].meta.shape[2]
        gi = graph.infer_shapes(g, 2)
        tg = autodiff.build_training_graph(gi)
        a = graph.infer_shapes(tg.graph, 2)
        b = graph.infer_shapes(passes.relu_mask_from_output(a), 2)
        assert any(n.op in ("ReluBack", "ReLU6Back") for n in b.nodes)
        for n in b.nodes:
            if n.op in ("ReluBack", "ReLU6Back"):
                assert b.find_node(n.inputs[1]).op in ("ReLU", "ReLU6")
        assert len(partition.partition(passes.run_pipeline(b))) < len(partition.partition(passes.run_pipeline(a)))
        rng = np.random.default_rng(1)
        ins = {"x": rng.uniform(-1, 1, (2, 3, hw, hw)).astype(np.float32)}
        t = np.zeros((2, 10), np.float32)
        t[np.arange(2), [3, 7]] = 1
        ins["t"] = t
        ea, eb = O.run_graph(a, ins), O.run_graph(b, ins)
        for _, gn in tg.param_grads:
            assert np.array_equal(ea[gn], eb[gn]), gn
