"""Graph IR mirror of the reference's model layer.

The B200 backend sits behind the reference's graph IR (``proj/include/sol/model.hpp``); this
module restates the parts the host side needs to drive it: op kinds, attrs, layer nodes, the
model DAG with Kahn ordering, shape inference, the JSON model schema and the SOLW weights
container, plus a seeded graph builder with the reference test builder's API.

Citations (reference = /root/reference/proj):
  * OpKind names / order            include/sol/model.hpp:24-57, src/model.cpp:22-53
  * Attrs defaults                  include/sol/model.hpp:64-80
  * validate_and_sort (Kahn)        src/model.cpp:107-170
  * infer_node_shape                src/model.cpp:203-352
  * model JSON schema               src/model_io.cpp:213-284 (parse_model_json / model_to_json)
  * SOLW container                  src/model_io.cpp:339-385
  * GraphBuilder init scales        tests/builders.hpp:33-164

Extensions beyond the reference IR (needed by BASELINE configs C5): ``Concat`` (along C0, any
arity) and ``ReLU6``. They are serialised with the same schema; the reference parser rejects
them, so their parity is checked against oracle/sol_oracle.py only ("parity unpinned").
"""
from __future__ import annotations

import copy
import dataclasses
import json
import math
import struct
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# --------------------------------------------------------------------------------------------
# Ops
# --------------------------------------------------------------------------------------------

# Names in the reference's kOps order (src/model.cpp:22-53) followed by our two extensions.
OP_NAMES = [
    "Conv2d", "Linear", "ReLU", "MaxPool2d", "AvgPool2d", "BatchNorm2d", "Add", "Flatten",
    "GlobalAvgPool", "Softmax", "CrossEntropyLoss", "Copy",
    "ReluBack", "MaxPool2dBack", "AvgPool2dBack", "GlobalAvgPoolBack", "FlattenBack",
    "SoftmaxBack", "SoftmaxCeBack", "CeBack", "BatchNormBackX", "BatchNormBackGamma",
    "BatchNormBackBeta", "Conv2dBackX", "Conv2dBackW", "Conv2dBackB", "LinearBackX",
    "LinearBackW", "LinearBackB", "SgdUpdate",
    # extensions (not in the reference IR)
    "Concat", "ReLU6", "ReLU6Back", "ConcatBack",
]
OP_ID = {n: i for i, n in enumerate(OP_NAMES)}
USER_FACING = set(OP_NAMES[:12]) | {"Concat", "ReLU6"}
EXTENSION_OPS = {"Concat", "ReLU6", "ReLU6Back", "ConcatBack"}


@dataclass
class Attrs:
    """Mirror of sol::Attrs (include/sol/model.hpp:64-80)."""
    out_channels: int = 0
    out_features: int = 0
    kh: int = 0
    kw: int = 0
    sh: int = 1
    sw: int = 1
    ph: int = 0
    pw: int = 0
    groups: int = 1
    has_bias: bool = True
    min_init: float = -math.inf
    count_padding: bool = False
    eps: float = 1e-5
    momentum: float = 0.1
    training: bool = False
    lr: float = 0.0
    # ConcatBack: channel offset of the slice
    offset: int = 0


# --------------------------------------------------------------------------------------------
# Tensor metas: canonical dim order only ([N0, C0, P1, P0] / [N0, C0] / [] / plain params)
# --------------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Meta:
    """Canonical tensor meta: kind is 'nchw', 'nc', 'scalar' or 'plain'."""
    kind: str
    shape: Tuple[int, ...]

    @property
    def numel(self) -> int:
        return int(np.prod(self.shape)) if self.shape else 1

    @property
    def n(self) -> int:
        return self.shape[0] if self.kind in ("nchw", "nc") else 1

    @property
    def c(self) -> int:
        if self.kind in ("nchw", "nc"):
            return self.shape[1]
        return self.shape[0] if self.kind == "plain" and len(self.shape) == 1 else 1

    @property
    def h(self) -> int:
        return self.shape[2] if self.kind == "nchw" else 1

    @property
    def w(self) -> int:
        return self.shape[3] if self.kind == "nchw" else 1

    def with_batch(self, b: int) -> "Meta":
        if self.kind in ("nchw", "nc") and self.shape[0] == 0:
            return Meta(self.kind, (b,) + self.shape[1:])
        return self

    def dims_json(self):
        """Reference JSON dims (src/model_io.cpp:45-52): extent 0 is the symbolic 'B'."""
        tags = {"nchw": [("N", 0), ("C", 0), ("P", 1), ("P", 0)], "nc": [("N", 0), ("C", 0)]}[self.kind]
        return [{"tag": t, "index": i, "extent": ("B" if e == 0 else int(e))}
                for (t, i), e in zip(tags, self.shape)]


def meta_nchw(n, c, h, w) -> Meta:
    return Meta("nchw", (n, c, h, w))


def meta_nc(n, c) -> Meta:
    return Meta("nc", (n, c))


def meta_plain(*extents) -> Meta:
    return Meta("plain", tuple(int(e) for e in extents))


SCALAR = Meta("scalar", ())


@dataclass
class LayerNode:
    id: str
    op: str
    attrs: Attrs = field(default_factory=Attrs)
    inputs: List[str] = field(default_factory=list)
    params: List[str] = field(default_factory=list)
    out_meta: Optional[Meta] = None
    saved_meta: Optional[Meta] = None


@dataclass
class GraphInput:
    name: str
    meta: Meta


class MalformedModelError(ValueError):
    pass


class ShapeMismatchError(ValueError):
    pass


@dataclass
class ModelGraph:
    graph_inputs: List[GraphInput] = field(default_factory=list)
    nodes: List[LayerNode] = field(default_factory=list)
    outputs: List[str] = field(default_factory=list)
    params: Dict[str, np.ndarray] = field(default_factory=dict)

    def copy(self) -> "ModelGraph":
        g = ModelGraph(copy.deepcopy(self.graph_inputs), copy.deepcopy(self.nodes),
                       list(self.outputs), dict(self.params))
        return g

    def find_node(self, nid: str) -> Optional[LayerNode]:
        idx = self.__dict__.get("_index")
        if idx is None or len(idx) != len(self.nodes):
            self.reindex()
            idx = self._index
        return idx.get(nid)

    def reindex(self):
        self._index = {n.id: n for n in self.nodes}

    def find_input(self, name: str) -> Optional[GraphInput]:
        for gi in self.graph_inputs:
            if gi.name == name:
                return gi
        return None

    def meta_of(self, name: str) -> Meta:
        gi = self.find_input(name)
        if gi is not None:
            return gi.meta
        n = self.find_node(name)
        if n is None or n.out_meta is None:
            raise MalformedModelError(f"no meta for tensor '{name}'")
        return n.out_meta

    def consumers(self) -> Dict[str, List[str]]:
        out: Dict[str, List[str]] = {}
        for n in self.nodes:
            for i in n.inputs:
                out.setdefault(i, []).append(n.id)
        return out

    # src/model.cpp:107-170
    def validate_and_sort(self) -> None:
        names = set()
        for gi in self.graph_inputs:
            if gi.name in names:
                raise MalformedModelError(f"duplicate graph input '{gi.name}'")
            names.add(gi.name)
        for n in self.nodes:
            if not n.id:
                raise MalformedModelError("node with empty id")
            if n.id in names:
                raise MalformedModelError(f"duplicate node id '{n.id}'")
            names.add(n.id)
        for n in self.nodes:
            for i in n.inputs:
                if i not in names:
                    raise MalformedModelError(f"node '{n.id}' references undefined input '{i}'")
            for p in n.params:
                if p not in self.params:
                    raise MalformedModelError(f"node '{n.id}' references missing parameter '{p}'")
            a = n.attrs
            if n.op == "Conv2d":
                if a.groups <= 0 or a.kh <= 0 or a.kw <= 0 or a.sh <= 0 or a.sw <= 0 or a.out_channels <= 0:
                    raise MalformedModelError(f"bad Conv2d attrs on '{n.id}'")
                if a.out_channels % a.groups:
                    raise MalformedModelError(f"Conv2d groups must divide out_channels on '{n.id}'")
                if a.ph >= a.kh or a.pw >= a.kw:
                    raise MalformedModelError(f"Conv2d padding must be smaller than kernel on '{n.id}'")
            if n.op in ("MaxPool2d", "AvgPool2d") and (a.kh <= 0 or a.kw <= 0 or a.ph >= a.kh or a.pw >= a.kw):
                raise MalformedModelError(f"bad pool attrs on '{n.id}'")
            if n.op == "Add" and len(n.inputs) != 2:
                raise MalformedModelError(f"Add expects 2 inputs on '{n.id}'")
            if n.op == "Concat" and len(n.inputs) < 1:
                raise MalformedModelError(f"Concat expects inputs on '{n.id}'")
        node_ids = {n.id for n in self.nodes}
        for o in self.outputs:
            if o not in node_ids:
                raise MalformedModelError(f"undeclared output node '{o}'")
        indeg = {n.id: 0 for n in self.nodes}
        succ: Dict[str, List[str]] = {}
        for n in self.nodes:
            for i in n.inputs:
                if i in node_ids:
                    indeg[n.id] += 1
                    succ.setdefault(i, []).append(n.id)
        by_id = {n.id: n for n in self.nodes}
        ready = [n.id for n in self.nodes if indeg[n.id] == 0]
        out = []
        head = 0
        while head < len(ready):
            nid = ready[head]
            head += 1
            out.append(by_id[nid])
            for s in succ.get(nid, []):
                indeg[s] -= 1
                if indeg[s] == 0:
                    ready.append(s)
        if len(out) != len(self.nodes):
            raise MalformedModelError("cycle in model graph")
        self.nodes = out
        self.reindex()


def _conv_out(i, k, s, p):
    return (i + 2 * p - k) // s + 1


def _req(cond, msg):
    if not cond:
        raise ShapeMismatchError(msg)


def infer_node_shape(n: LayerNode, ins: Sequence[Meta]) -> Meta:
    """src/model.cpp:203-352 (+ Concat / ReLU6 extensions)."""
    a = n.attrs
    op = n.op
    if op == "Conv2d":
        x = ins[0]
        _req(x.kind == "nchw", f"Conv2d expects pixel dims on '{n.id}'")
        _req(x.c % a.groups == 0, f"Conv2d groups must divide in-channels on '{n.id}'")
        return meta_nchw(x.n, a.out_channels, _conv_out(x.h, a.kh, a.sh, a.ph), _conv_out(x.w, a.kw, a.sw, a.pw))
    if op in ("MaxPool2d", "AvgPool2d"):
        x = ins[0]
        return meta_nchw(x.n, x.c, _conv_out(x.h, a.kh, a.sh, a.ph), _conv_out(x.w, a.kw, a.sw, a.pw))
    if op == "Linear":
        x = ins[0]
        _req(x.kind == "nc", f"Linear expects a [batch, channel] tensor on '{n.id}'")
        return meta_nc(x.n, a.out_features)
    if op in ("ReLU", "ReLU6", "Copy", "BatchNorm2d", "Softmax"):
        return ins[0]
    if op == "Add":
        _req(ins[0] == ins[1], f"Add operands differ on '{n.id}'")
        return ins[0]
    if op == "Concat":
        x = ins[0]
        for m in ins[1:]:
            _req(m.kind == x.kind and m.n == x.n and m.h == x.h and m.w == x.w, f"Concat mismatch on '{n.id}'")
        c = sum(m.c for m in ins)
        return meta_nchw(x.n, c, x.h, x.w) if x.kind == "nchw" else meta_nc(x.n, c)
    if op == "Flatten":
        x = ins[0]
        return meta_nc(x.n, x.numel // x.n)
    if op == "GlobalAvgPool":
        x = ins[0]
        return meta_nc(x.n, x.c)
    if op == "CrossEntropyLoss":
        _req(ins[0].numel == ins[1].numel, "CrossEntropyLoss prediction/label mismatch")
        return SCALAR
    if op in ("ReluBack", "ReLU6Back", "MaxPool2dBack", "SoftmaxBack", "BatchNormBackX"):
        return ins[1]
    if op in ("AvgPool2dBack", "GlobalAvgPoolBack", "FlattenBack", "Conv2dBackX", "LinearBackX",
              "Conv2dBackW", "Conv2dBackB", "LinearBackW", "LinearBackB", "ConcatBack"):
        _req(n.saved_meta is not None, f"{op} needs saved meta")
        return n.saved_meta
    if op in ("SoftmaxCeBack", "CeBack"):
        return ins[0]
    if op in ("BatchNormBackGamma", "BatchNormBackBeta"):
        return meta_plain(ins[0].c)
    if op == "SgdUpdate":
        return ins[0]
    raise ShapeMismatchError(f"no shape rule for op {op}")


def infer_shapes(g: ModelGraph, batch: int) -> ModelGraph:
    """src/model.cpp:375-392: substitutes the symbolic batch and annotates every node."""
    _req(batch > 0, "batch must be positive")
    out = g.copy()
    for gi in out.graph_inputs:
        gi.meta = gi.meta.with_batch(batch)
    metas = {gi.name: gi.meta for gi in out.graph_inputs}
    for n in out.nodes:
        n.out_meta = infer_node_shape(n, [metas[i] for i in n.inputs])
        metas[n.id] = n.out_meta
    out.reindex()
    return out


# --------------------------------------------------------------------------------------------
# Serialisation: reference model JSON + SOLW weights
# --------------------------------------------------------------------------------------------

def _attrs_json(n: LayerNode) -> dict:
    a = n.attrs
    j: dict = {}
    if a.training:
        j["training"] = True
    if n.op == "Conv2d":
        j.update(out_channels=a.out_channels, kernel=[a.kh, a.kw], stride=[a.sh, a.sw],
                 padding=[a.ph, a.pw], groups=a.groups, bias=a.has_bias)
    elif n.op == "Linear":
        j.update(out_features=a.out_features, bias=a.has_bias)
    elif n.op == "MaxPool2d":
        j.update(kernel=[a.kh, a.kw], stride=[a.sh, a.sw], padding=[a.ph, a.pw])
        if not math.isinf(a.min_init):
            j["min_init"] = a.min_init
    elif n.op == "AvgPool2d":
        j.update(kernel=[a.kh, a.kw], stride=[a.sh, a.sw], padding=[a.ph, a.pw],
                 count_padding=a.count_padding)
    elif n.op == "BatchNorm2d":
        j.update(eps=a.eps, momentum=a.momentum)
    return j


def model_to_json(g: ModelGraph) -> str:
    """Reference model schema (src/model_io.cpp:213-284)."""
    j = {
        "inputs": [{"name": gi.name, "dims": gi.meta.dims_json()} for gi in g.graph_inputs],
        "nodes": [{"id": n.id, "op": n.op, "attrs": _attrs_json(n), "inputs": list(n.inputs),
                   "params": list(n.params)} for n in g.nodes],
        "outputs": list(g.outputs),
    }
    return json.dumps(j)


def _pair(v):
    return (int(v), int(v)) if isinstance(v, (int, float)) else (int(v[0]), int(v[1]))


def model_from_json(text: str, weights: Optional[bytes] = None) -> ModelGraph:
    """Parses the reference model schema (src/model_io.cpp:213-260, attrs :60-100) and binds
    SOLW weights; validates and topologically sorts like load_model (:287-294)."""
    j = json.loads(text)
    g = ModelGraph()
    for inp in j["inputs"]:
        tags = [(d["tag"], d["index"]) for d in inp["dims"]]
        ext = tuple(0 if d["extent"] == "B" else int(d["extent"]) for d in inp["dims"])
        kind = "nchw" if tags == [("N", 0), ("C", 0), ("P", 1), ("P", 0)] else \
            "nc" if tags == [("N", 0), ("C", 0)] else None
        if kind is None:
            raise MalformedModelError(f"unsupported input dims {tags}")
        g.graph_inputs.append(GraphInput(inp["name"], Meta(kind, ext)))
    for nj in j["nodes"]:
        op = nj["op"]
        if op not in USER_FACING:
            raise MalformedModelError(f"unsupported op '{op}'")
        aj = nj.get("attrs", {})
        a = Attrs()
        if op == "Conv2d":
            a.out_channels = int(aj["out_channels"])
            a.kh, a.kw = _pair(aj["kernel"])
            a.sh, a.sw = _pair(aj.get("stride", 1))
            a.ph, a.pw = _pair(aj.get("padding", 0))
            a.groups = int(aj.get("groups", 1))
            a.has_bias = bool(aj.get("bias", True))
        elif op == "Linear":
            a.out_features = int(aj["out_features"])
            a.has_bias = bool(aj.get("bias", True))
        elif op in ("MaxPool2d", "AvgPool2d"):
            a.kh, a.kw = _pair(aj["kernel"])
            a.sh, a.sw = _pair(aj.get("stride", [a.kh, a.kw]))   # stride defaults to kernel (:82)
            a.ph, a.pw = _pair(aj.get("padding", 0))
            if op == "MaxPool2d":
                a.min_init = float(aj.get("min_init", -math.inf))
            else:
                a.count_padding = bool(aj.get("count_padding", False))
        elif op == "BatchNorm2d":
            a.eps = float(aj.get("eps", 1e-5))
            a.momentum = float(aj.get("momentum", 0.1))
        a.training = bool(aj.get("training", False))
        g.nodes.append(LayerNode(nj["id"], op, a, list(nj.get("inputs", [])), list(nj.get("params", []))))
    g.outputs = list(j["outputs"])
    if weights is not None:
        g.params = weights_from_bytes(weights)
    g.validate_and_sort()
    return g


def weights_to_bytes(params: Dict[str, np.ndarray]) -> bytes:
    """SOLW v1 (src/model_io.cpp:339-364): name-sorted, u16 name len, u8 dtype, u8 rank, u32 dims."""
    out = bytearray(b"SOLW")
    out += struct.pack("<II", 1, len(params))
    for name in sorted(params):
        t = np.ascontiguousarray(params[name])
        f64 = t.dtype == np.float64
        t = t if f64 else t.astype(np.float32)
        nb = name.encode()
        out += struct.pack("<H", len(nb)) + nb
        out += struct.pack("<BB", 1 if f64 else 0, t.ndim)
        out += struct.pack("<%dI" % t.ndim, *t.shape)
        out += t.tobytes()
    return bytes(out)


def weights_from_bytes(b: bytes) -> Dict[str, np.ndarray]:
    if b[:4] != b"SOLW":
        raise ValueError("bad weights magic")
    ver, count = struct.unpack_from("<II", b, 4)
    if ver != 1:
        raise ValueError(f"unsupported weights version {ver}")
    pos = 12
    out = {}
    for _ in range(count):
        (ln,) = struct.unpack_from("<H", b, pos)
        pos += 2
        name = b[pos:pos + ln].decode()
        pos += ln
        dt, nd = struct.unpack_from("<BB", b, pos)
        pos += 2
        shape = struct.unpack_from("<%dI" % nd, b, pos)
        pos += 4 * nd
        dtype = np.float64 if dt == 1 else np.float32
        cnt = int(np.prod(shape)) if shape else 1
        out[name] = np.frombuffer(b, dtype=dtype, count=cnt, offset=pos).reshape(shape).copy()
        pos += cnt * np.dtype(dtype).itemsize
    if pos != len(b):
        raise ValueError("trailing bytes in weights file")
    return out


# --------------------------------------------------------------------------------------------
# Builder (tests/builders.hpp:33-164 API, numpy-seeded)
# --------------------------------------------------------------------------------------------

class GraphBuilder:
    """Builds graphs with the reference test builder's API and init distributions:
    conv/linear U(+-1/sqrt(fan_in)); BN gamma U(0.5,1.5), beta U(-0.5,0.5),
    running mean U(-0.5,0.5), running var U(0.5,1.5)."""

    def __init__(self, seed: int = 1):
        self.g = ModelGraph()
        self.rng = np.random.default_rng(seed)

    def input(self, name: str, meta: Meta) -> str:
        self.g.graph_inputs.append(GraphInput(name, meta))
        return name

    def _init(self, shape, scale):
        return self.rng.uniform(-scale, scale, size=shape).astype(np.float32)

    def node(self, nid, op, inputs, attrs=None, params=None) -> str:
        self.g.nodes.append(LayerNode(nid, op, attrs or Attrs(), list(inputs), list(params or [])))
        return nid

    def conv(self, nid, x, in_c, out_c, k, s=1, p=0, groups=1, bias=True) -> str:
        a = Attrs(out_channels=out_c, kh=k, kw=k, sh=s, sw=s, ph=p, pw=p, groups=groups, has_bias=bias)
        scale = 1.0 / math.sqrt(in_c // groups * k * k)
        self.g.params[nid + ".W"] = self._init((out_c, in_c // groups, k, k), scale)
        ps = [nid + ".W"]
        if bias:
            self.g.params[nid + ".b"] = self._init((out_c,), scale)
            ps.append(nid + ".b")
        return self.node(nid, "Conv2d", [x], a, ps)

    def linear(self, nid, x, in_f, out_f, bias=True) -> str:
        a = Attrs(out_features=out_f, has_bias=bias)
        scale = 1.0 / math.sqrt(in_f)
        self.g.params[nid + ".W"] = self._init((out_f, in_f), scale)
        ps = [nid + ".W"]
        if bias:
            self.g.params[nid + ".b"] = self._init((out_f,), scale)
            ps.append(nid + ".b")
        return self.node(nid, "Linear", [x], a, ps)

    def relu(self, nid, x):
        return self.node(nid, "ReLU", [x])

    def relu6(self, nid, x):
        return self.node(nid, "ReLU6", [x])

    def maxpool(self, nid, x, k, s=0, p=0):
        return self.node(nid, "MaxPool2d", [x], Attrs(kh=k, kw=k, sh=s or k, sw=s or k, ph=p, pw=p))

    def avgpool(self, nid, x, k, s=0, p=0, count_padding=False):
        return self.node(nid, "AvgPool2d", [x], Attrs(kh=k, kw=k, sh=s or k, sw=s or k, ph=p, pw=p,
                                                       count_padding=count_padding))

    def batchnorm(self, nid, x, c, training=False):
        r = self.rng
        self.g.params[nid + ".gamma"] = r.uniform(0.5, 1.5, c).astype(np.float32)
        self.g.params[nid + ".beta"] = (r.uniform(0.5, 1.5, c) - 1.0).astype(np.float32)
        self.g.params[nid + ".running_mean"] = (r.uniform(0.5, 1.5, c) - 1.0).astype(np.float32)
        self.g.params[nid + ".running_var"] = r.uniform(0.5, 1.5, c).astype(np.float32)
        return self.node(nid, "BatchNorm2d", [x], Attrs(training=training),
                         [nid + ".gamma", nid + ".beta", nid + ".running_mean", nid + ".running_var"])

    def flatten(self, nid, x):
        return self.node(nid, "Flatten", [x])

    def softmax(self, nid, x):
        return self.node(nid, "Softmax", [x])

    def add(self, nid, a, b):
        return self.node(nid, "Add", [a, b])

    def concat(self, nid, xs):
        return self.node(nid, "Concat", list(xs))

    def gap(self, nid, x):
        return self.node(nid, "GlobalAvgPool", [x])

    def ce(self, nid, pred, labels):
        return self.node(nid, "CrossEntropyLoss", [pred, labels])

    def done(self, outputs) -> ModelGraph:
        self.g.outputs = list(outputs)
        self.g.validate_and_sort()
        return self.g


def uses_extensions(g: ModelGraph) -> bool:
    return any(n.op in EXTENSION_OPS for n in g.nodes)
