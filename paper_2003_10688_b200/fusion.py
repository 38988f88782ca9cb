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


def _ops(g: ModelGraph, u: ExecUnit):
    return [g.find_node(i).op for i in u.node_ids]


def _is_1x1(n, stride_one: bool) -> bool:
    a = n.attrs
    return (a.kh == 1 and a.kw == 1 and a.ph == 0 and a.pw == 0 and a.groups <= 1 and a.sh == a.sw
            and (a.sh == 1 or not stride_one))


def fuse_bottleneck_tails(g: ModelGraph, units: List[ExecUnit], block: int = 64) -> List[ExecUnit]:
    """Merges a fused [Conv1x1, BN, Add, ReLU] unit with the fused [Conv1x1(stride s), BN] unit that
    produces its residual (ResNet bottleneck tail + downsample) into ONE dual-GEMM unit
    [conv, bn, conv_ds, bn_ds, add, relu]: both BN scales fold into the weights, the downsample
    output never touches HBM. Needs both conv inputs in 128-byte channel blocks (`block`)."""
    cons = g.consumers()
    outputs = set(g.outputs)
    by_out = {u.output: i for i, u in enumerate(units)}
    drop, repl = set(), {}
    for j, v in enumerate(units):
        if v.kind != "dnn":
            continue
        ops = _ops(g, v)
        if ops[:3] != ["Conv2d", "BatchNorm2d", "Add"] or len(ops) not in (3, 4):
            continue
        if len(ops) == 4 and ops[3] not in ("ReLU", "ReLU6"):
            continue
        conv = g.find_node(v.node_ids[0])
        add = g.find_node(v.node_ids[2])
        res = add.inputs[1] if add.inputs[0] == v.node_ids[1] else add.inputs[0]
        i = by_out.get(res)
        if i is None or i in drop:
            continue
        u = units[i]
        if u.kind != "dnn" or _ops(g, u) != ["Conv2d", "BatchNorm2d"] or res in outputs:
            continue
        if len(cons.get(res, [])) != 1:
            continue
        ds = g.find_node(u.node_ids[0])
        if not (_is_1x1(conv, True) and _is_1x1(ds, False)):
            continue
        c_main = g.meta_of(conv.inputs[0]).shape[1]
        c_ds = g.meta_of(ds.inputs[0]).shape[1]
        if c_main % block or c_ds % block:
            continue
        node_ids = list(v.node_ids[:2]) + list(u.node_ids) + list(v.node_ids[2:])
        inputs = [x for x in v.inputs if x != res] + [x for x in u.inputs if x not in v.inputs]
        params = list(v.params) + [p for p in u.params if p not in v.params]
        repl[j] = ExecUnit("dnn", node_ids, v.output, inputs, params)
        drop.add(i)
    return [repl.get(j, w) for j, w in enumerate(units) if j not in drop]


def fuse_stem_pool(g: ModelGraph, units: List[ExecUnit], direct_inputs) -> List[ExecUnit]:
    """Merges the stride-2 stem conv (reading a canonical NCHW graph input, see
    frontend._direct_stem_inputs) with its single consumer DFP unit
    [BatchNorm2d(inference)] [-> ReLU] -> MaxPool2d(3x3, stride 2, pad 1) into ONE heavy unit
    [Conv2d, BN, (ReLU), MaxPool2d]: the stem kernel (stem_row.cu) folds the BN into its epilogue and
    max-pools its own output rows in shared memory, so the full-resolution activation (4x the pooled
    tensor) is never written or re-read. MaxPool2d's min_init (0 after the relu-into-pool pass,
    passes.cpp:76-102) is the pool's initial value, as in the reference lowering."""
    cons = g.consumers()
    outputs = set(g.outputs)
    owner = {nid: i for i, u in enumerate(units) for nid in u.node_ids}
    drop, repl = set(), {}
    for i, u in enumerate(units):
        if u.kind != "dnn" or _ops(g, u) != ["Conv2d"]:
            continue
        conv = g.find_node(u.node_ids[0])
        a = conv.attrs
        if conv.inputs[0] not in direct_inputs or a.sh != 2 or a.sw != 2 or a.kw > 8 or a.groups > 1:
            continue
        _, cout, oh, ow = g.meta_of(conv.id).shape
        if cout != 64 or oh % 2 or ow % 2 or ow > 124 or u.output in outputs:
            continue
        c = cons.get(u.output, [])
        if len(c) != 1:
            continue
        j = owner[c[0]]
        v = units[j]
        ops = _ops(g, v)
        if v.kind != "dfp" or v.node_ids[0] != c[0] or ops not in (["BatchNorm2d", "MaxPool2d"],
                                                                   ["BatchNorm2d", "ReLU", "MaxPool2d"]):
            continue
        nodes = [g.find_node(n) for n in v.node_ids]
        if nodes[0].attrs.training or nodes[0].inputs[0] != u.output:
            continue
        if any(nodes[k].inputs[0] != nodes[k - 1].id for k in range(1, len(nodes))):
            continue
        p = nodes[-1].attrs
        if (p.kh, p.kw, p.sh, p.sw, p.ph, p.pw) != (3, 3, 2, 2, 1, 1):
            continue
        inputs = list(u.inputs) + [x for x in v.inputs if x != u.output and x not in u.inputs]
        params = list(u.params) + [q for q in v.params if q not in u.params]
        repl[j] = ExecUnit("dnn", list(u.node_ids) + list(v.node_ids), v.output, inputs, params)
        drop.add(i)
    return [repl.get(j, w) for j, w in enumerate(units) if j not in drop]


def fuse_dgrad_relu_back(g: ModelGraph, units: List[ExecUnit]) -> List[ExecUnit]:
    """Training plans: a stride-1 Conv2dBackX unit whose output feeds exactly one unit
      ReluBack(dx, relu_out)                  (inner ReLUs), or
      Add(dx, g) -> ReluBack(sum, relu_out)   (block outputs: dx from the next block's conv1,
                                               g the skip-path gradient)
    with the mask read from the ReLU output (passes.relu_mask_from_output) is merged with it: the
    dgrad GEMM epilogue writes relu_out > 0 ? [bf16(dx) + g | dx] : 0, bit-for-bit the separate
    unit's output (the epilogue rounds dx to the stored precision before the add, as the unfused
    plan does), and dx never round-trips through HBM (a write and two reads of an activation-sized
    tensor per ReLU saved). The merged unit runs at the consumer's position. Strided dgrads
    (sub-pixel classes + interleave) and grouped convs keep the separate unit."""
    cons = g.consumers()
    outputs = set(g.outputs)
    owner = {}
    for i, u in enumerate(units):
        for nid in u.node_ids:
            owner[nid] = i
    merged_into = {}
    for i, u in enumerate(units):
        if u.kind != "dnn" or len(u.node_ids) != 1:
            continue
        n = g.find_node(u.output)
        a = n.attrs
        if n.op != "Conv2dBackX" or a.groups > 1 or max(a.sh, 1) != 1 or max(a.sw, 1) != 1:
            continue
        c = cons.get(u.output, [])
        if len(c) != 1 or u.output in outputs:
            continue
        j = owner[c[0]]
        v = units[j]
        if v.kind != "dfp" or len(v.node_ids) > 2 or j in merged_into.values():
            continue
        vn = [g.find_node(n) for n in v.node_ids]
        r = vn[-1]
        if r.op != "ReluBack" or len(r.inputs) != 2 or len(vn) > 2:
            continue
        if g.find_node(r.inputs[1]) is None or g.find_node(r.inputs[1]).op != "ReLU":
            continue  # the mask must be a ReLU output (relu_mask_from_output)
        if len(vn) == 1:  # ReluBack(dx, relu_out)
            if r.inputs[0] != u.output or r.inputs[1] == u.output:
                continue
        else:  # Add(dx, g) -> ReluBack(sum, relu_out): the block-output gradient
            ad = vn[0]
            if ad.op != "Add" or len(ad.inputs) != 2 or u.output not in ad.inputs or r.inputs[0] != ad.id:
                continue
            other = ad.inputs[1] if ad.inputs[0] == u.output else ad.inputs[0]
            if other == u.output or other not in v.inputs or r.inputs[1] == u.output:
                continue
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
        out.append(ExecUnit("dnn", list(u.node_ids) + list(v.node_ids), v.output, inputs, list(u.params)))
    return out

