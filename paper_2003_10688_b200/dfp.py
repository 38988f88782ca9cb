"""Module compile boundary: an ExecUnit of the partitioned graph -> a B200 kernel module.

Mirrors the reference's `lower_group(graph, unit, flavor, overrides) -> KernelIR` and
`interpret(KernelIR, inputs, output)` contract (include/sol/dfp.hpp:43-58): the unit's member ops,
attrs and boundary bindings (activations first, then params — KernelIR input order,
src/dfp_lower.cpp:931-939) cross the C ABI as a `sol_unit_desc`; the library selects a
hand-written sm_100a kernel family (or a tcgen05 provider for heavy nodes) and returns a module.
An unknown op signature is a compile-time error (SOL_E_UNSUPPORTED) — there is no fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Dict, List, Optional

from . import _lib as L
from .graph import OP_ID, Meta, ModelGraph
from .partition import ExecUnit

DTYPES = {"f32": L.DT_F32, "bf16": L.DT_BF16}
ELEM = {L.DT_F32: 4, L.DT_BF16: 2}

# ops that are internal plan steps (the reference's Step::Kind::Reorder, frontend.hpp:41-50)
OP_REORDER_IN = 100   # canonical NCHW/NC f32 host layout -> NHWC plan storage
OP_REORDER_OUT = 101  # NHWC plan storage -> canonical f32


def vec_of(dtype: int) -> int:
    return 16 // ELEM[dtype]


def storage_ld(meta: Meta, dtype: int) -> int:
    """Row stride (elements) of an activation in plan storage: channels padded to 16 bytes."""
    if meta.kind == "scalar":
        return 1
    c = meta.c
    v = vec_of(dtype)
    return (c + v - 1) // v * v


def storage_bytes(meta: Meta, dtype: int, f32: bool = False) -> int:
    es = 4 if f32 else ELEM[dtype]
    if meta.kind == "scalar":
        return es
    if meta.kind == "plain":
        return 4 * meta.numel
    pix = meta.numel // meta.c
    return pix * storage_ld(meta, dtype) * es


def _dims(meta: Meta, arr):
    for i in range(4):
        arr[i] = 0
    for i, e in enumerate(meta.shape[:4]):
        arr[i] = int(e)
    return len(meta.shape)


def binding_for(meta: Meta, dtype: int, is_param: bool, f32: bool = False) -> L.Binding:
    b = L.Binding()
    is_param = is_param or meta.kind == "plain"   # plain f32 tensors: params and their gradients
    b.is_param = int(is_param)
    b.dtype = L.DT_F32 if (is_param or f32) else dtype
    b.rank = _dims(meta, b.dims)
    b.ld = 0 if is_param or meta.kind == "scalar" else storage_ld(meta, dtype)
    return b


# outputs stored as f32 regardless of the plan dtype (loss, parameter gradients)
F32_OUTPUT_OPS = {"CrossEntropyLoss", "BatchNormBackGamma", "BatchNormBackBeta", "Conv2dBackW",
                  "Conv2dBackB", "LinearBackW", "LinearBackB", "SgdUpdate"}


def is_f32_tensor(g: ModelGraph, name: str) -> bool:
    n = g.find_node(name)
    return n is not None and n.op in F32_OUTPUT_OPS


@dataclass
class UnitModule:
    handle: C.c_void_p
    family: str
    n_args: int
    scratch_bytes: int
    algo_bytes: float
    algo_flops: float
    launches: int
    launches_frozen: int = -1  # -1: same as launches

    def __post_init__(self):
        if self.launches_frozen < 0:
            self.launches_frozen = self.launches

    def info(self):
        return dict(family=self.family, algo_bytes=self.algo_bytes, algo_flops=self.algo_flops)


def _attrs(a) -> L.Attrs:
    x = L.Attrs()
    x.out_channels = a.out_channels
    x.out_features = a.out_features
    x.kh, x.kw, x.sh, x.sw, x.ph, x.pw = a.kh, a.kw, a.sh, a.sw, a.ph, a.pw
    x.groups = a.groups
    x.has_bias = int(a.has_bias)
    x.min_init = a.min_init
    x.count_padding = int(a.count_padding)
    x.eps = a.eps
    x.momentum = a.momentum
    x.training = int(a.training)
    x.lr = a.lr
    x.offset = a.offset
    return x


def build_desc(g: ModelGraph, unit: ExecUnit, dtype: int, nchw_inputs=()):
    """sol_unit_desc for a unit of shape-inferred graph `g` (keeps the ctypes arrays alive).
    Names in `nchw_inputs` are bound in the canonical host layout (NCHW f32, is_param = 2)."""
    names = list(unit.inputs) + list(unit.params)
    index = {n: i for i, n in enumerate(names)}
    bindings = (L.Binding * max(1, len(names)))()
    for i, nm in enumerate(names):
        if nm in g.params:
            bindings[i] = binding_for(Meta("plain", tuple(g.params[nm].shape)), dtype, True)
        elif nm in nchw_inputs:
            b = binding_for(g.meta_of(nm), dtype, False)
            b.is_param = 2
            b.dtype = L.DT_F32
            b.ld = g.meta_of(nm).shape[1]
            bindings[i] = b
        else:
            bindings[i] = binding_for(g.meta_of(nm), dtype, False, is_f32_tensor(g, nm))
    pos = {nid: k for k, nid in enumerate(unit.node_ids)}
    ops = (L.UnitOp * len(unit.node_ids))()
    for k, nid in enumerate(unit.node_ids):
        n = g.find_node(nid)
        o = ops[k]
        o.op = OP_ID[n.op]
        if len(n.inputs) > L.MAX_OP_IN:
            raise L.UnsupportedError(L.SOL_E_UNSUPPORTED, f"{n.op} arity {len(n.inputs)}")
        o.n_inputs = len(n.inputs)
        for i, inp in enumerate(n.inputs):
            o.inputs[i] = -(pos[inp] + 1) if inp in pos else index[inp]
        o.n_params = len(n.params)
        for i, p in enumerate(n.params):
            o.params[i] = index[p]
        o.attrs = _attrs(n.attrs)
        o.saved_rank = _dims(n.saved_meta, o.saved_dims) if n.saved_meta is not None else 0
        o.out_rank = _dims(n.out_meta, o.out_dims)
    d = L.UnitDesc()
    d.kind = 1 if unit.kind == "dnn" else 0
    d.n_ops = len(unit.node_ids)
    d.ops = C.cast(ops, C.POINTER(L.UnitOp))
    d.n_bindings = len(names)
    d.bindings = C.cast(bindings, C.POINTER(L.Binding))
    d.output = binding_for(g.meta_of(unit.output), dtype, False, is_f32_tensor(g, unit.output))
    d.dtype = dtype
    return d, (ops, bindings)


def create_module(g: ModelGraph, unit: ExecUnit, dtype: int, nchw_inputs=()) -> UnitModule:
    d, keep = build_desc(g, unit, dtype, nchw_inputs)
    h = C.c_void_p()
    L.check(L.lib().sol_b200_module_create(C.byref(d), C.byref(h)))
    info = L.ModuleInfo()
    L.check(L.lib().sol_b200_module_info(h, C.byref(info)))
    return UnitModule(h, info.family.decode(), info.n_args, info.scratch_bytes, info.algo_bytes,
                      info.algo_flops, info.launches, info.launches_frozen)


def reorder_module(meta: Meta, dtype: int, inbound: bool) -> UnitModule:
    """Step::Kind::Reorder: canonical f32 <-> NHWC plan storage for a graph input / output."""
    ops = (L.UnitOp * 1)()
    o = ops[0]
    o.op = OP_REORDER_IN if inbound else OP_REORDER_OUT
    o.n_inputs = 1
    o.inputs[0] = 0
    o.out_rank = _dims(meta, o.out_dims)
    bindings = (L.Binding * 1)()
    canon = L.Binding()
    canon.is_param = 0
    canon.dtype = L.DT_F32
    canon.rank = _dims(meta, canon.dims)
    canon.ld = meta.c if meta.kind != "scalar" else 1
    stored = binding_for(meta, dtype, False)
    d = L.UnitDesc()
    d.kind = 0
    d.n_ops = 1
    d.ops = C.cast(ops, C.POINTER(L.UnitOp))
    d.n_bindings = 1
    bindings[0] = canon if inbound else stored
    d.bindings = C.cast(bindings, C.POINTER(L.Binding))
    d.output = stored if inbound else canon
    d.dtype = dtype
    h = C.c_void_p()
    L.check(L.lib().sol_b200_module_create(C.byref(d), C.byref(h)))
    info = L.ModuleInfo()
    L.check(L.lib().sol_b200_module_info(h, C.byref(info)))
    return UnitModule(h, info.family.decode(), info.n_args, info.scratch_bytes, info.algo_bytes,
                      info.algo_flops, info.launches, info.launches_frozen)


def sgd_multi_module(shapes, lr: float, dtype: int) -> UnitModule:
    """All SgdUpdate units of a training plan as ONE module (one multi-tensor launch): bindings are
    (param, grad) pairs, updates are in place; the unit output aliases the first parameter."""
    n = len(shapes)
    ops = (L.UnitOp * n)()
    bindings = (L.Binding * (2 * n))()
    for i, shape in enumerate(shapes):
        o = ops[i]
        o.op = OP_ID["SgdUpdate"]
        o.n_inputs = 2
        o.inputs[0] = 2 * i
        o.inputs[1] = 2 * i + 1
        o.attrs = L.Attrs()
        o.attrs.lr = lr
        meta = Meta("plain", tuple(shape))
        o.out_rank = _dims(meta, o.out_dims)
        bindings[2 * i] = binding_for(meta, dtype, True)
        bindings[2 * i + 1] = binding_for(meta, dtype, True)
    d = L.UnitDesc()
    d.kind = 0
    d.n_ops = n
    d.ops = C.cast(ops, C.POINTER(L.UnitOp))
    d.n_bindings = 2 * n
    d.bindings = C.cast(bindings, C.POINTER(L.Binding))
    d.output = binding_for(Meta("plain", tuple(shapes[0])), dtype, True)
    d.dtype = dtype
    h = C.c_void_p()
    L.check(L.lib().sol_b200_module_create(C.byref(d), C.byref(h)))
    info = L.ModuleInfo()
    L.check(L.lib().sol_b200_module_info(h, C.byref(info)))
    return UnitModule(h, info.family.decode(), info.n_args, info.scratch_bytes, info.algo_bytes,
                      info.algo_flops, info.launches, info.launches_frozen)


def sgd_module(shape, lr: float, dtype: int) -> UnitModule:
    """SgdUpdate unit (dfp_lower.cpp:780-783) over a parameter and its gradient (f32)."""
    ops = (L.UnitOp * 1)()
    o = ops[0]
    o.op = OP_ID["SgdUpdate"]
    o.n_inputs = 2
    o.inputs[0] = 0
    o.inputs[1] = 1
    o.attrs = L.Attrs()
    o.attrs.lr = lr
    meta = Meta("plain", tuple(shape))
    o.out_rank = _dims(meta, o.out_dims)
    bindings = (L.Binding * 2)()
    bindings[0] = binding_for(meta, dtype, True)
    bindings[1] = binding_for(meta, dtype, True)
    d = L.UnitDesc()
    d.kind = 0
    d.n_ops = 1
    d.ops = C.cast(ops, C.POINTER(L.UnitOp))
    d.n_bindings = 2
    d.bindings = C.cast(bindings, C.POINTER(L.Binding))
    d.output = binding_for(meta, dtype, True)
    d.dtype = dtype
    h = C.c_void_p()
    L.check(L.lib().sol_b200_module_create(C.byref(d), C.byref(h)))
    info = L.ModuleInfo()
    L.check(L.lib().sol_b200_module_info(h, C.byref(info)))
    return UnitModule(h, info.family.decode(), info.n_args, info.scratch_bytes, info.algo_bytes,
                      info.algo_flops, info.launches, info.launches_frozen)
