"""Reverse-mode training graph, mirroring the reference autodiff.

  * build_backward           src/autodiff.cpp:75-228 (fused SoftmaxCeBack :94-101, pruning :202-214)
  * build_training_graph     src/autodiff.cpp:230-249 (BN switched to batch statistics)
  * grad accumulation names  src/autodiff.cpp:58-71 ("d_<t>_acc<k>" Add chains)
Extensions: ReLU6 -> ReLU6Back, Concat -> one ConcatBack (channel slice) per input.
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

from .graph import Attrs, GraphInput, LayerNode, ModelGraph, infer_shapes, meta_plain


class NonDifferentiableGraphError(ValueError):
    pass


@dataclass
class TrainingGraph:
    graph: ModelGraph
    loss: str
    param_grads: List[Tuple[str, str]] = field(default_factory=list)


def _build_backward(g: ModelGraph):
    if len(g.outputs) != 1:
        raise NonDifferentiableGraphError("expected a single loss output")
    loss = g.find_node(g.outputs[0])
    if loss is None or loss.op != "CrossEntropyLoss":
        raise NonDifferentiableGraphError("graph does not end in CrossEntropyLoss")
    bw = ModelGraph(params=g.params)
    contributions: Dict[str, List[str]] = {}
    saved: List[str] = []
    saved_set = set()
    param_grads: List[Tuple[str, str]] = []

    def use_fwd(name):
        if name not in saved_set:
            saved_set.add(name)
            saved.append(name)
            bw.graph_inputs.append(GraphInput(name, g.meta_of(name)))
        return name

    def emit(nid, op, inputs, attrs, params=(), saved_meta=None):
        bw.nodes.append(LayerNode(nid, op, copy.copy(attrs), list(inputs), list(params), None, saved_meta))
        return nid

    def contribute(t, grad):
        if g.find_node(t) is not None or g.find_input(t) is not None:
            contributions.setdefault(t, []).append(grad)

    def grad_of(t):
        lst = contributions.get(t)
        if not lst:
            return ""
        while len(lst) > 1:
            a, b = lst[0], lst[1]
            nid = f"d_{t}_acc{len(lst)}"
            emit(nid, "Add", [a, b], Attrs())
            del lst[:2]
            lst.insert(0, nid)
        return lst[0]

    cons = g.consumers()
    pred, labels = loss.inputs[0], loss.inputs[1]
    pn = g.find_node(pred)
    skip = {loss.id}
    if pn is not None and pn.op == "Softmax" and len(cons[pred]) == 1 and pred not in g.outputs:
        nid = emit("d_" + pn.inputs[0], "SoftmaxCeBack", [use_fwd(pred), use_fwd(labels)], Attrs())
        contribute(pn.inputs[0], nid)
        skip.add(pn.id)
    else:
        nid = emit("d_" + pred, "CeBack", [use_fwd(pred), use_fwd(labels)], Attrs())
        contribute(pred, nid)

    for n in reversed(g.nodes):
        if n.id in skip:
            continue
        delta = grad_of(n.id)
        if not delta:
            continue
        x = n.inputs[0] if n.inputs else ""
        a = n.attrs
        via = lambda t: f"d_{t}_via_{n.id}"
        if n.op == "ReLU":
            contribute(x, emit(via(x), "ReluBack", [delta, use_fwd(x)], a))
        elif n.op == "ReLU6":
            contribute(x, emit(via(x), "ReLU6Back", [delta, use_fwd(x)], a))
        elif n.op == "Copy":
            contribute(x, delta)
        elif n.op == "Add":
            contribute(n.inputs[0], delta)
            contribute(n.inputs[1], delta)
        elif n.op == "Concat":
            off = 0
            for t in n.inputs:
                m = g.meta_of(t)
                aa = Attrs(offset=off)
                contribute(t, emit(via(t), "ConcatBack", [delta], aa, (), m))
                off += m.c
        elif n.op == "MaxPool2d":
            contribute(x, emit(via(x), "MaxPool2dBack", [delta, use_fwd(x)], a))
        elif n.op == "AvgPool2d":
            contribute(x, emit(via(x), "AvgPool2dBack", [delta], a, (), g.meta_of(x)))
        elif n.op == "GlobalAvgPool":
            contribute(x, emit(via(x), "GlobalAvgPoolBack", [delta], a, (), g.meta_of(x)))
        elif n.op == "Flatten":
            contribute(x, emit(via(x), "FlattenBack", [delta], a, (), g.meta_of(x)))
        elif n.op == "Softmax":
            contribute(x, emit(via(x), "SoftmaxBack", [delta, use_fwd(n.id)], a))
        elif n.op == "BatchNorm2d":
            x_params = [n.params[0]]
            gamma_params = []
            if not a.training:
                x_params = [n.params[0], n.params[2], n.params[3]]
                gamma_params = [n.params[2], n.params[3]]
            contribute(x, emit(via(x), "BatchNormBackX", [delta, use_fwd(x)], a, x_params))
            param_grads.append((n.params[0], emit("g_" + n.params[0], "BatchNormBackGamma",
                                                  [delta, use_fwd(x)], a, gamma_params)))
            param_grads.append((n.params[1], emit("g_" + n.params[1], "BatchNormBackBeta", [delta], a)))
        elif n.op == "Conv2d":
            if g.find_node(x) is not None:
                contribute(x, emit(via(x), "Conv2dBackX", [delta], a, [n.params[0]], g.meta_of(x)))
            param_grads.append((n.params[0], emit("g_" + n.params[0], "Conv2dBackW",
                                                  [delta, use_fwd(x)], a, (),
                                                  meta_plain(*g.params[n.params[0]].shape))))
            if a.has_bias:
                param_grads.append((n.params[1], emit("g_" + n.params[1], "Conv2dBackB", [delta], a,
                                                      (), meta_plain(*g.params[n.params[1]].shape))))
        elif n.op == "Linear":
            if g.find_node(x) is not None:
                contribute(x, emit(via(x), "LinearBackX", [delta], a, [n.params[0]], g.meta_of(x)))
            param_grads.append((n.params[0], emit("g_" + n.params[0], "LinearBackW",
                                                  [delta, use_fwd(x)], a, (),
                                                  meta_plain(*g.params[n.params[0]].shape))))
            if a.has_bias:
                param_grads.append((n.params[1], emit("g_" + n.params[1], "LinearBackB", [delta], a,
                                                      (), meta_plain(*g.params[n.params[1]].shape))))
        else:
            raise NonDifferentiableGraphError(f"no gradient rule for {n.op}")

    # prune nodes not feeding a parameter gradient (autodiff.cpp:202-214)
    needed = set()
    stack = [nid for _, nid in param_grads]
    bw_ids = {n.id for n in bw.nodes}
    by_id = {n.id: n for n in bw.nodes}
    while stack:
        nid = stack.pop()
        if nid in needed:
            continue
        needed.add(nid)
        if nid in by_id:
            for i in by_id[nid].inputs:
                if i in bw_ids:
                    stack.append(i)
    bw.nodes = [n for n in bw.nodes if n.id in needed]
    param_grads.sort()
    bw.outputs = [nid for _, nid in param_grads]
    bw.validate_and_sort()
    batch = next((gi.meta.n for gi in g.graph_inputs if gi.meta.kind in ("nchw", "nc")), 1)
    return infer_shapes(bw, batch), param_grads, saved


def build_training_graph(g: ModelGraph) -> TrainingGraph:
    """Forward (BN in batch-statistics mode) + backward in one graph; outputs [loss, grads...]."""
    fwd = g.copy()
    for n in fwd.nodes:
        if n.op == "BatchNorm2d":
            n.attrs.training = True
    bwg, param_grads, _ = _build_backward(fwd)
    out = fwd.copy()
    out.nodes = out.nodes + bwg.nodes
    out.outputs = [fwd.outputs[0]] + [nid for _, nid in param_grads]
    out.validate_and_sort()
    return TrainingGraph(out, fwd.outputs[0], param_grads)
