"""Execution-unit partition, mirroring the reference DFP partitioner.

  * ExecUnit                   include/sol/dfp.hpp:21-28
  * group_breaker (Flatten)    src/dfp_lower.cpp:23
  * is_depthwise_conv          src/dfp_lower.cpp:27-31 (groups == Cout == Cin)
  * heavy_in_graph             src/dfp_lower.cpp:33-54
  * partition / join rule      src/dfp_lower.cpp:70-165, :91-103

The units are the work list the B200 executor runs: every DnnNode goes to a tcgen05 provider
kernel and every DfpGroup to one hand-written fused sm_100a kernel selected by its op signature.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

from .graph import LayerNode, ModelGraph


@dataclass
class ExecUnit:
    kind: str                       # "dfp" | "dnn"
    node_ids: List[str] = field(default_factory=list)
    output: str = ""
    inputs: List[str] = field(default_factory=list)   # external activations, first-use order
    params: List[str] = field(default_factory=list)   # parameter names, first-use order


def is_depthwise_conv(n: LayerNode, cin: int) -> bool:
    return (n.op == "Conv2d" and n.attrs.groups > 1 and n.attrs.groups == n.attrs.out_channels
            and n.attrs.groups == cin)


def heavy_in_graph(g: ModelGraph, n: LayerNode) -> bool:
    a = n.attrs
    if n.op in ("Linear", "LinearBackX", "LinearBackW"):
        return True
    if n.op == "Conv2d":
        return not is_depthwise_conv(n, g.meta_of(n.inputs[0]).c)
    if n.op == "Conv2dBackX":
        cin = n.saved_meta.c if n.saved_meta is not None else -1
        return not (a.groups > 1 and a.groups == a.out_channels and a.groups == cin)
    if n.op == "Conv2dBackW":
        icg = n.saved_meta.shape[1] if n.saved_meta is not None and len(n.saved_meta.shape) == 4 else -1
        return not (a.groups > 1 and a.groups == a.out_channels and icg == 1)
    return False


def _breaker(op: str) -> bool:
    return op == "Flatten"


def partition(g: ModelGraph) -> List[ExecUnit]:
    cons = g.consumers()
    outputs = set(g.outputs)
    groups: List[dict] = []
    group_of = {}
    order = []  # [last node pos, handle]; handle >= 0 group, < 0 heavy node index

    def join_ok(grp, n):
        if grp["breaker"] or _breaker(n.op):
            return False
        inside = set(grp["members"]) | {n.id}
        for m in grp["members"]:
            if m in outputs or m not in cons:
                return False
            if any(c not in inside for c in cons[m]):
                return False
        return True

    for i, n in enumerate(g.nodes):
        if heavy_in_graph(g, n):
            order.append([i, -i - 1])
            continue
        joined = -1
        for inp in n.inputs:
            gi = group_of.get(inp)
            if gi is None:
                continue
            if join_ok(groups[gi], n):
                joined = gi
                break
        if joined < 0:
            groups.append({"members": [n.id], "breaker": _breaker(n.op)})
            joined = len(groups) - 1
            order.append([i, joined])
        else:
            groups[joined]["members"].append(n.id)
            for o in order:
                if o[1] == joined:
                    o[0] = i
        group_of[n.id] = joined

    order.sort(key=lambda o: o[0])  # stable, as std::stable_sort
    units = []
    for _, h in order:
        if h < 0:
            n = g.nodes[-h - 1]
            units.append(ExecUnit("dnn", [n.id], n.id, list(n.inputs), list(n.params)))
        else:
            members = groups[h]["members"]
            inside = set(members)
            u = ExecUnit("dfp", list(members), members[-1])
            for mid in members:
                m = g.find_node(mid)
                for inp in m.inputs:
                    if inp not in inside and inp not in u.inputs:
                        u.inputs.append(inp)
                for p in m.params:
                    if p not in u.params:
                        u.params.append(p)
            units.append(u)
    return units
