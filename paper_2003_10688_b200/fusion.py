"""Plan-level epilogue fusion ("Epilogue fusion / BN folding ... beyond the
reference's pass set, keep it behind a flag with oracle parity").

For inference plans, a heavy Conv2d/Linear unit whose output feeds exactly one DFP unit of the
form  BatchNorm2d(inference) [-> Add(residual)] [-> ReLU | ReLU6]  is merged with it: the tcgen05
GEMM epilogue applies the folded BN scale/shift, adds the residual tile and clamps, so the conv
output never round-trips through HBM. Unit outputs that remain are bit-for-bit the same tensors
(modulo one fewer bf16 rounding), and the executed unit order is unchanged.
"""
from __future__ import annotations

from typing import List

from .graph import ModelGraph
from .partition import ExecUnit


def _chain_ok(g: ModelGraph, v: ExecUnit, conv_out: str) -> bool:
    ops = [g.find_node(i) for i in v.node_ids]
    k = 0
    prev = conv_out
    if k < len(ops) and ops[k].op == "BatchNorm2d":
        if ops[k].attrs.training or ops[k].inputs[0] != prev:
            return False
        prev = ops[k].id
        k += 1
    else:
        return False
    if k < len(ops) and ops[k].op == "Add":
        a, b = ops[k].inputs
        other = b if a == prev else (a if b == prev else None)
        if other is None or other not in v.inputs:
            return False
        prev = ops[k].id
        k += 1
    if k < len(ops) and ops[k].op in ("ReLU", "ReLU6"):
        if ops[k].inputs[0] != prev:
            return False
        k += 1
    return k == len(ops)


def fuse_conv_epilogues(g: ModelGraph, units: List[ExecUnit]) -> List[ExecUnit]:
    cons = g.consumers()
    outputs = set(g.outputs)
    owner = {}
    for i, u in enumerate(units):
        for nid in u.node_ids:
            owner[nid] = i
    merged_into = {}
    for i, u in enumerate(units):
        if u.kind != "dnn" or g.find_node(u.output).op not in ("Conv2d", "Linear"):
            continue
        c = cons.get(u.output, [])
        if len(c) != 1 or u.output in outputs:
            continue
        j = owner[c[0]]
        v = units[j]
        if v.kind != "dfp" or v.node_ids[0] != c[0] or j in merged_into.values():
            continue
        if _chain_ok(g, v, u.output):
            merged_into[i] = j
    out = []
    absorbed = set(merged_into)
    for j, v in enumerate(units):
        if j in absorbed:
            continue
        src = [i for i, jj in merged_into.items() if jj == j]
        if not src:
            out.append(v)
            continue
        u = units[src[0]]
        inputs = list(u.inputs) + [x for x in v.inputs if x != u.output and x not in u.inputs]
        params = list(u.params) + [p for p in v.params if p not in u.params]
        out.append(ExecUnit("dnn", list(u.node_ids) + list(v.node_ids), v.output, inputs, params))
    return out
