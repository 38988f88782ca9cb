#!/usr/bin/env python3
"""Generates tests/golden/* from the REFERENCE itself (oracle/_ref/libsolref.so, compiled from the
unmodified sources under /root/reference/proj/src by oracle/Makefile). Run in the build container:

    make -C oracle && python scripts/make_golden.py

Fixtures (small, committed):
  * <case>.npz   : model JSON + SOLW weights + inputs + every node output of the reference's f64
                   oracle run_reference (reference.cpp:589-605), canonical layout, f32
  * partition_<case>.json : the reference partition (dfp_lower.cpp:70-165) after its pass pipeline
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refbridge  # noqa: E402
from paper_2003_10688_b200 import autodiff, graph, models  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def inputs_for(g, batch, seed):
    rng = np.random.default_rng(seed)
    ins = {}
    for gi in g.graph_inputs:
        shape = (batch,) + gi.meta.shape[1:]
        if gi.name == "t":
            t = np.zeros(shape, np.float32)
            t[np.arange(batch), np.arange(batch) % shape[1]] = 1.0
            ins["t"] = t
        else:
            ins[gi.name] = rng.uniform(-1, 1, shape).astype(np.float32)
    return ins


def make_case(name, g, batch, training=False, seed=0):
    mj, wb = graph.model_to_json(g), graph.weights_to_bytes(g.params)
    s = refbridge.RefSession(mj, wb, batch, training)
    ins = inputs_for(g, batch, seed)
    for k, v in ins.items():
        s.set_input(k, v)
    s.run_reference()
    gj = s.graph_json()
    outs = {}
    for n in gj["nodes"]:
        outs["out/" + n["id"]] = s.get(n["id"])
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), model_json=np.frombuffer(mj.encode(), np.uint8),
                        weights=np.frombuffer(wb, np.uint8), batch=np.int64(batch), training=np.int64(training),
                        **{"in/" + k: v for k, v in ins.items()}, **outs)
    print(name, len(outs), "node outputs")


def make_partition(name, g, batch, training=False):
    s = refbridge.RefSession(graph.model_to_json(g), graph.weights_to_bytes(g.params), batch, training)
    s.pipeline()
    with open(os.path.join(OUT, f"partition_{name}.json"), "w") as f:
        json.dump({"units": s.partition(), "graph": s.graph_json(),
                   "param_grads": s.param_grads() if training else []}, f)
    print("partition", name)


def main():
    os.makedirs(OUT, exist_ok=True)
    refbridge.build()
    make_case("small_cnn_infer", models.small_cnn(hw=16), 2)
    make_case("small_cnn_train", models.small_cnn(hw=16, train=True), 4, training=True)
    make_case("resnet18_tiny_infer", models.resnet(18, hw=32, classes=10, width=8), 2)
    make_case("resnet50_tiny_train", models.resnet(50, hw=32, classes=10, width=8, train=True), 2, training=True)
    make_partition("resnet50", models.resnet(50), 2)
    make_partition("resnet50_train", models.resnet(50, train=True), 2, training=True)
    make_partition("resnet18", models.resnet(18), 2)
    make_partition("small_cnn", models.small_cnn(), 2)
    make_partition("small_cnn_train", models.small_cnn(train=True), 2, training=True)


if __name__ == "__main__":
    main()
