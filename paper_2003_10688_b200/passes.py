"""Exact-math graph rewrites, mirroring the reference pass pipeline.

  * fuse_relu_pool     src/passes.cpp:76-102, :150-156  (ReLU adjacent to MaxPool2d -> min_init=0)
  * reorder_commuting  src/passes.cpp:107-149, :158-163 (ReLU commutes past Flatten toward a pool)
  * run_pipeline       src/passes.cpp:168-178           (alternate to fixpoint)
"""
from __future__ import annotations

from .graph import ModelGraph


def _remove_node(g: ModelGraph, victim: str, replacement: str) -> None:
    for n in g.nodes:
        n.inputs = [replacement if i == victim else i for i in n.inputs]
    g.outputs = [replacement if o == victim else o for o in g.outputs]
    g.nodes = [n for n in g.nodes if n.id != victim]
    g.reindex()


def _fuse_one(g: ModelGraph) -> bool:
    cons = g.consumers()
    outs = set(g.outputs)
    for n in g.nodes:
        if n.op == "ReLU":
            c = cons.get(n.id, [])
            if len(c) != 1 or n.id in outs:
                continue
            pool = g.find_node(c[0])
            if pool is None or pool.op != "MaxPool2d":
                continue
            pool.attrs.min_init = max(pool.attrs.min_init, 0.0)
            _remove_node(g, n.id, n.inputs[0])
            return True
        if n.op == "MaxPool2d":
            c = cons.get(n.id, [])
            if len(c) != 1 or n.id in outs:
                continue
            relu = g.find_node(c[0])
            if relu is None or relu.op != "ReLU":
                continue
            n.attrs.min_init = max(n.attrs.min_init, 0.0)
            _remove_node(g, relu.id, n.id)
            return True
    return False


def _reorder_one(g: ModelGraph) -> bool:
    cons = g.consumers()
    outs = set(g.outputs)

    def sole(nid):
        c = cons.get(nid, [])
        return g.find_node(c[0]) if len(c) == 1 else None

    for n in g.nodes:
        if n.op != "MaxPool2d" or n.id in outs:
            continue
        chain = []
        cur = n
        while True:
            nxt = sole(cur.id)
            if nxt is None:
                break
            if nxt.op == "ReLU" and chain:
                shape_node = g.find_node(chain[-1])
                relu = nxt
                upstream = shape_node.inputs[0]
                relu.inputs[0] = upstream
                shape_node.inputs[0] = relu.id
                for m in g.nodes:
                    if m.id == shape_node.id:
                        continue
                    m.inputs = [shape_node.id if i == relu.id else i for i in m.inputs]
                g.outputs = [shape_node.id if o == relu.id else o for o in g.outputs]
                if relu.out_meta is not None:
                    relu.out_meta = g.meta_of(upstream)
                g.validate_and_sort()
                return True
            if nxt.op != "Flatten" or nxt.id in outs:
                break
            chain.append(nxt.id)
            cur = nxt
    return False


def fuse_relu_pool(g: ModelGraph) -> ModelGraph:
    out = g.copy()
    while _fuse_one(out):
        pass
    out.validate_and_sort()
    return out


def reorder_commuting(g: ModelGraph) -> ModelGraph:
    out = g.copy()
    while _reorder_one(out):
        pass
    return out


def _fingerprint(g: ModelGraph):
    return tuple((n.id, n.op, tuple(n.inputs), n.attrs.min_init) for n in g.nodes) + tuple(g.outputs)


def run_pipeline(g: ModelGraph) -> ModelGraph:
    cur = g
    while True:
        before = _fingerprint(cur)
        cur = fuse_relu_pool(reorder_commuting(cur))
        if _fingerprint(cur) == before:
            return cur


def relu_mask_from_output(g: ModelGraph) -> ModelGraph:
    """Training-graph rewrite beyond the reference pass set (plan option `relu_mask_from_output`):
    ReluBack(delta, x) -> ReluBack(delta, relu(x)) and ReLU6Back(delta, x) -> ReLU6Back(delta,
    relu6(x)). Exact: x > 0 <=> relu(x) > 0 and 0 < x < 6 <=> 0 < relu6(x) < 6 (also after bf16
    rounding, which preserves sign and order). The pre-activation then has the activation as its
    only consumer, so partition() fuses BN [+ Add] + ReLU into one unit that never writes the
    pre-activation tensor (one full activation write per BN saved in the forward pass)."""
    g = g.copy()
    by_input = {}
    for n in g.nodes:
        if n.op in ("ReLU", "ReLU6") and n.inputs:
            by_input.setdefault((n.op, n.inputs[0]), n.id)
    for n in g.nodes:
        if n.op in ("ReluBack", "ReLU6Back") and len(n.inputs) == 2:
            fwd = by_input.get(("ReLU" if n.op == "ReluBack" else "ReLU6", n.inputs[1]))
            if fwd is not None:
                n.inputs = [n.inputs[0], fwd]
    g.reindex()
    return g
