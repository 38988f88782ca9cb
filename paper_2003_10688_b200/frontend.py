"""Network API over the B200 backend: optimize() -> OptimizedModel.predict / train_step.

This is the frontend the reference declares but does not implement
(include/sol/frontend.hpp:104-174: fe::optimize, OptimizedModel::predict, train_step(batch, lr,
TrainMode::Native), load_state, DevicePlan/Step). The compile pipeline follows the declared one
(frontend.hpp:167-172): infer_shapes -> [build_training_graph] -> run_pipeline -> partition ->
per-unit module compile -> plan (buffers + steps) -> layouts. The plan executes in C++
(libsolb200.so: arena placement by liveness, one CUDA stream, optional CUDA-graph replay, NCCL
all-reduce of gradients for batch-sharded data parallelism) — Python only compiles.

Activations live in NHWC (ActLayout::ChannelsLast) in the plan dtype (bf16, or f32 with TF32
tensor-core GEMMs); parameters are f32 master copies in the reference's canonical layouts.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import hashlib
import json
import os
import threading
import time
import weakref
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _lib as L
from .autodiff import build_training_graph
from .dfp import (DTYPES, ELEM, create_module, is_f32_tensor, reorder_module, sgd_module, sgd_multi_module,
                  storage_bytes)
from .dp import allreduce_schedule
from .graph import Meta, ModelGraph, infer_shapes
from .partition import ExecUnit, partition
from .passes import run_pipeline


@dataclass
class OptimizeOptions:
    """Mirror of fe::OptimizeOptions (frontend.hpp:27-36) plus the B200 knobs."""
    batch: int = 1
    dtype: str = "bf16"        # "bf16" or "f32" (TF32 tensor cores, f32 storage)
    train: bool = False        # compile forward+backward+SGD (TrainMode::Native)
    lr: float = 0.1
    use_graph: bool = True     # replay the plan as one CUDA graph
    device: int = 0
    world_size: int = 1        # batch-sharded data parallelism (one process per GPU)
    rank: int = 0
    nccl_id: Optional[bytes] = None
    passes: bool = True        # reference rewrite pipeline (passes.cpp:168-178)
    keep_all: bool = False     # debug: every unit output persistent (no arena reuse)
    fuse_epilogue: bool = False  # inference: fold BN(+Add)(+ReLU) units into the conv epilogue
    fuse_bn_backward: bool = True  # training: BatchNormBackX also writes its Gamma/Beta siblings
    multi_sgd: bool = True         # training: every SgdUpdate in one multi-tensor launch
    nccl_allreduce: bool = False   # test hook: run the NCCL gradient all-reduce even with one replica
    relu_mask_from_output: bool = True  # training: ReluBack masks read the ReLU output (passes.py), so
                                        # BN+ReLU fuse and the pre-activation is never stored
    bn_stats_from_conv: bool = True  # training, bf16: a training BN's batch statistics come out of the
                                     # producing conv's GEMM epilogue (no statistics pass over its output)
    fuse_relu_back: bool = True    # training: a stride-1 Conv2dBackX applies the following ReluBack
                                   # mask (read from the ReLU output) in its GEMM epilogue
    update_bn_stats: bool = True   # training: update BN running_mean / running_var on the device
                                   # (autodiff::update_bn_running_stats, autodiff.cpp:356-384)
    autotune: bool = False         # measure the tcgen05 tile configs of every conv/linear (dnn.cpp:214-290)
    tune_budget: int = 5           # measured runs per candidate (median; one warm-up besides)
    tune_cache_path: Optional[str] = None  # persistent TuneCache JSON (None: process-wide, in memory)
    cache: bool = True             # optimize() returns the live model compiled for the same graph+options

    def fingerprint(self) -> str:
        """fe::OptimizeOptions::fingerprint (frontend.hpp:35): every field that changes the plan."""
        d = {k: v for k, v in self.__dict__.items() if k not in ("nccl_id", "tune_cache_path", "cache")}
        d["env"] = sorted((k, v) for k, v in os.environ.items() if k.startswith("SOL_"))
        return json.dumps(d, sort_keys=True, default=str)


@dataclass
class StepInfo:
    kind: str          # "unit" | "reorder" | "sgd" | "allreduce"
    family: str
    output: str
    algo_bytes: float = 0.0
    algo_flops: float = 0.0
    launches: int = 1
    launches_frozen: int = 1  # once the plan is frozen (inference: cached weight packing)
    node_ids: List[str] = field(default_factory=list)


_COPY_POOL = None


def parallel_copy(dst: np.ndarray, src: np.ndarray):
    """dst[...] = src split over host threads along the batch dimension (numpy releases the GIL
    for plain copies): filling a 154 MB pinned batch single-threaded costs ~4x one B200 step."""
    global _COPY_POOL
    n = dst.shape[0] if dst.ndim else 1
    if dst.nbytes < (8 << 20) or n < 2:
        np.copyto(dst, src)
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1)))
    parts = min(n, _COPY_POOL._max_workers * 2)
    bounds = [(i * n // parts, (i + 1) * n // parts) for i in range(parts)]
    list(_COPY_POOL.map(lambda b: np.copyto(dst[b[0]:b[1]], src[b[0]:b[1]]), bounds))


class PinnedBuffer:
    """Page-locked host memory (cudaMallocHost through the C ABI) viewed as a numpy array."""

    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        L.check(L.lib().sol_b200_host_alloc(max(nbytes, 16), C.byref(self.ptr)))
        self.nbytes = nbytes
        buf = (C.c_uint8 * max(nbytes, 16)).from_address(self.ptr.value)
        self.u8 = np.frombuffer(buf, dtype=np.uint8)

    def view(self, dtype, shape):
        n = int(np.prod(shape)) if shape else 1
        return self.u8[: n * np.dtype(dtype).itemsize].view(dtype).reshape(shape)

    def __del__(self):
        try:
            if self.ptr:
                L.lib().sol_b200_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DevicePlan:
    """One compiled plan on one device (fe::DevicePlan / Step, frontend.hpp:41-61): the compiled
    graph, its units, one plan buffer per tensor, one step per unit module, optionally the gradient
    all-reduce buckets and the SGD step; executed by libsolb200 (eagerly, or replayed as a CUDA
    graph). OptimizedModel owns one per mode (forward, training)."""

    def __init__(self, g: ModelGraph, options: OptimizeOptions):
        t0 = time.perf_counter()
        self.options = options
        self.dtype = DTYPES[options.dtype]
        gi = infer_shapes(g, options.batch)
        self.param_grads = []
        if options.train:
            tg = build_training_graph(gi)
            cg = infer_shapes(tg.graph, options.batch)
            self.loss_name = tg.loss
            self.param_grads = list(tg.param_grads)
        else:
            cg = gi
            self.loss_name = None
        if options.train and options.relu_mask_from_output:
            from .passes import relu_mask_from_output
            cg = infer_shapes(relu_mask_from_output(cg), options.batch)
        if options.passes:
            cg = run_pipeline(cg)
        self.graph = cg
        self.units: List[ExecUnit] = partition(cg)
        if (options.train and options.relu_mask_from_output and options.fuse_relu_back
                and not os.environ.get("SOL_NO_FUSE_RELU_BACK")):
            from .fusion import fuse_dgrad_relu_back
            self.units = fuse_dgrad_relu_back(cg, self.units)
        if options.fuse_epilogue and not options.train:
            from .fusion import fuse_bottleneck_tails, fuse_conv_epilogues
            self.units = fuse_conv_epilogues(cg, self.units)
            # dual-GEMM bottleneck tails (kill switch SOL_NO_DUAL=1)
            if options.dtype == "bf16" and not os.environ.get("SOL_NO_DUAL"):
                self.units = fuse_bottleneck_tails(cg, self.units)
            # stem conv + BN + 3x3/2 max pool in one kernel: exact, but still slower than the
            # unfused pair (284 us vs 166 + 95 us on B200; 8 epilogue warps measured 298 us), so
            # opt-in only
            if os.environ.get("SOL_STEM_POOL"):
                from .fusion import fuse_stem_pool
                self.units = fuse_stem_pool(cg, self.units, self._direct_stem_inputs())
        self.params: Dict[str, np.ndarray] = {k: np.asarray(v, np.float32).copy() for k, v in g.params.items()}
        self._build_plan()
        self.lr = options.lr
        self.tuner_runs, self.tune_cache_hits, self.tuned = 0, 0, {}
        self.compile_ms = (time.perf_counter() - t0) * 1e3

    # ------------------------------------------------------------------------------------------
    def _build_plan(self):
        o = self.options
        lib = L.lib()
        self.plan = C.c_void_p()
        L.check(lib.sol_b200_plan_create(o.device, C.byref(self.plan)))
        g = self.graph
        self.buf: Dict[str, int] = {}
        self.steps: List[StepInfo] = []
        self._step_ids: List[List[int]] = []

        def add_buf(nbytes, persistent):
            i = C.c_int32()
            L.check(lib.sol_b200_plan_add_buffer(self.plan, int(nbytes), int(persistent), C.byref(i)))
            return i.value

        def add_step(mod, ids, info: StepInfo):
            arr = (C.c_int32 * len(ids))(*ids)
            L.check(lib.sol_b200_plan_add_step(self.plan, mod.handle, arr, len(ids)))
            info.family = mod.family
            info.algo_bytes, info.algo_flops, info.launches = mod.algo_bytes, mod.algo_flops, mod.launches
            info.launches_frozen = getattr(mod, "launches_frozen", mod.launches)
            self.steps.append(info)

        # parameters: persistent f32 master copies
        for name, arr in self.params.items():
            self.buf[name] = add_buf(arr.nbytes, True)
        outputs = set(g.outputs)
        # graph inputs: canonical f32 staging buffer + NHWC plan buffer + reorder step
        self.inputs: Dict[str, Meta] = {}
        self.in_canon: Dict[str, int] = {}
        direct = self._direct_stem_inputs()
        for gi in g.graph_inputs:
            self.inputs[gi.name] = gi.meta
            self.in_canon[gi.name] = add_buf(4 * gi.meta.numel, True)
            if gi.name in direct:
                # the stem conv reads the canonical NCHW f32 buffer itself (no reorder pass)
                self.buf[gi.name] = self.in_canon[gi.name]
                continue
            self.buf[gi.name] = add_buf(storage_bytes(gi.meta, self.dtype), True)
            add_step(reorder_module(gi.meta, self.dtype, True), [self.in_canon[gi.name], self.buf[gi.name]],
                     StepInfo("reorder", "", gi.name))
        # unit outputs
        self.modules = []
        siblings = bn_back_siblings(g, self.units) if (o.train and o.fuse_bn_backward) else {}
        absorbed = {v for sib in siblings.values() for v in sib if v is not None}
        act_sibs = activation_siblings(g, self.units) if o.fuse_bn_backward else {}
        absorbed |= {v[0] for v in act_sibs.values()}

        def out_buf(name):
            if name not in self.buf:
                meta = g.meta_of(name)
                self.buf[name] = add_buf(storage_bytes(meta, self.dtype, is_f32_tensor(g, name)),
                                         name in outputs or o.keep_all)
            return self.buf[name]

        # gradient all-reduce buckets: a bucket is issued right after the unit that
        # completes its last gradient, so NCCL (on the plan's comm stream) overlaps the remaining
        # backward units; ~25 MB buckets (SOL_AR_BUCKET_MB). The schedule is dp.allreduce_schedule.
        reduce_grads = o.train and (o.world_size > 1 or o.nccl_allreduce)
        self.ar_schedule = {}
        if reduce_grads:
            self.ar_schedule = allreduce_schedule(
                gradient_completions(self.units, siblings, absorbed),
                {gname: 4.0 * self.params[pname].size for pname, gname in self.param_grads},
                float(os.environ.get("SOL_AR_BUCKET_MB", "25")) * 2 ** 20)
        self.ar_buckets = len(self.ar_schedule)
        grad_param = {gname: pname for pname, gname in self.param_grads}

        def issue_bucket(names):
            for gname in names:
                n = self.params[grad_param[gname]].size
                L.check(lib.sol_b200_plan_add_allreduce(self.plan, self.buf[gname], n, L.DT_F32, 1.0 / o.world_size))
                self.steps.append(StepInfo("allreduce", "nccl_allreduce", gname, algo_bytes=4.0 * n))

        link_stats = (o.train and o.bn_stats_from_conv and o.dtype == "bf16"
                      and not os.environ.get("SOL_NO_BN_STATS_EPI"))
        conv_step = {}  # output of a single-Conv2d unit -> its plan step
        self.bn_stats_links = 0
        for ui, u in enumerate(self.units):
            out_buf(u.output)
            if u.output in absorbed:  # computed by its BatchNormBackX sibling's step
                issue_bucket(self.ar_schedule.get(ui, ()))
                continue
            mod = create_module(g, u, self.dtype, [n for n in u.inputs if n in direct])
            if o.train and o.update_bn_stats and any(
                    g.find_node(n).op == "BatchNorm2d" and g.find_node(n).attrs.training for n in u.node_ids):
                L.check(lib.sol_b200_module_set_option(mod.handle, L.MODOPT_UPDATE_BN_RUNNING_STATS, 1))
            ids = [self.buf[n] for n in list(u.inputs) + list(u.params)] + [self.buf[u.output]]
            if u.output in act_sibs:
                relu_out, mask = act_sibs[u.output]
                L.check(lib.sol_b200_module_set_sibling_outputs(mod.handle, mask))
                mod.n_args += 1
                ids += [out_buf(relu_out)]
            if u.output in siblings:
                gam, bet = siblings[u.output]
                mask = (1 if gam else 0) | (2 if bet else 0)
                L.check(lib.sol_b200_module_set_sibling_outputs(mod.handle, mask))
                mod.n_args += bin(mask).count("1")
                ids += [out_buf(x) for x in (gam, bet) if x]
            step = len(self.steps)
            add_step(mod, ids, StepInfo("unit", "", u.output, node_ids=list(u.node_ids)))
            if link_stats:
                first = g.find_node(u.node_ids[0])
                if u.kind == "dnn" and len(u.node_ids) == 1 and first.op == "Conv2d":
                    conv_step[u.output] = step
                elif (u.kind == "dfp" and first.op == "BatchNorm2d" and first.attrs.training
                      and first.inputs[0] in conv_step and first.inputs[0] in u.inputs):
                    rc = lib.sol_b200_plan_link_bn_stats(self.plan, conv_step[first.inputs[0]], step,
                                                         u.inputs.index(first.inputs[0]))
                    if rc == 0:
                        self.bn_stats_links += 1
                        self.steps[conv_step[first.inputs[0]]].family = "conv_fprop_bnstats_tcgen05"
                    elif rc != L.SOL_E_UNSUPPORTED:
                        L.check(rc)
            issue_bucket(self.ar_schedule.get(ui, ()))
        # graph outputs: canonical f32 copies for the host
        self.out_canon: Dict[str, int] = {}
        for name in g.outputs:
            meta = g.meta_of(name)
            if is_f32_tensor(g, name):
                self.out_canon[name] = self.buf[name]   # already canonical f32 (loss / gradients)
                continue
            self.out_canon[name] = add_buf(4 * meta.numel, True)
            add_step(reorder_module(meta, self.dtype, False), [self.buf[name], self.out_canon[name]],
                     StepInfo("reorder", "", name))
        # native training: all-reduce gradients across ranks, then SGD on the device
        if o.train:
            if o.multi_sgd and self.param_grads:
                for k in range(0, len(self.param_grads), 512):
                    chunk = self.param_grads[k:k + 512]
                    mod = sgd_multi_module([self.params[p].shape for p, _ in chunk], o.lr, self.dtype)
                    ids = [i for p, gname in chunk for i in (self.buf[p], self.buf[gname])] + [self.buf[chunk[0][0]]]
                    add_step(mod, ids, StepInfo("sgd", "", chunk[0][0]))
            else:
                for pname, gname in self.param_grads:
                    mod = sgd_module(self.params[pname].shape, o.lr, self.dtype)
                    add_step(mod, [self.buf[pname], self.buf[gname], self.buf[pname]], StepInfo("sgd", "", pname))
        if o.world_size > 1 or (o.train and o.nccl_allreduce):
            if o.nccl_id is None and o.world_size == 1:
                o.nccl_id = nccl_unique_id()
            if o.nccl_id is None:
                raise ValueError("world_size > 1 needs the rank-0 NCCL unique id")
            idb = (C.c_uint8 * 128)(*o.nccl_id)
            L.check(lib.sol_b200_plan_set_comm(self.plan, idb, o.rank, o.world_size))
        L.check(lib.sol_b200_plan_finalize(self.plan))
        self._upload_params()
        self._ran = False
        self.stream = C.c_void_p()
        L.check(lib.sol_b200_plan_stream(self.plan, C.byref(self.stream)))
        # pinned staging for the host interface
        self.pin_in = {n: [PinnedBuffer(4 * m.numel) for _ in range(2)] for n, m in self.inputs.items()}
        self._slot, self._slot_ticket = 0, [None, None]
        self.pin_out = {n: PinnedBuffer(4 * g.meta_of(n).numel) for n in g.outputs}

    def _direct_stem_inputs(self):
        """Graph inputs whose only consumer is a few-channel (<= 4) stem Conv2d unit in a bf16
        inference plan: that conv's halo loads read the canonical NCHW f32 input directly."""
        g, o = self.graph, self.options
        if o.dtype != "bf16" or o.train or os.environ.get("SOL_NO_DIRECT_STEM"):
            return set()
        out = set()
        for gi in g.graph_inputs:
            users = [u for u in self.units if gi.name in u.inputs]
            if len(users) != 1 or gi.meta.kind != "nchw" or gi.meta.shape[1] > 4:
                continue
            u = users[0]
            n0 = g.find_node(u.node_ids[0])
            if (u.kind == "dnn" and n0.op == "Conv2d" and n0.inputs[0] == gi.name and n0.attrs.groups <= 1
                    and n0.attrs.out_channels == 64 and n0.attrs.kw <= 8 and n0.attrs.kh * 32 <= 256
                    and sum(1 for n in u.node_ids for i in g.find_node(n).inputs if i == gi.name) == 1):
                out.add(gi.name)
        return out

    def _upload_params(self, names=None):
        """Host master parameters -> plan buffers (one pinned staging area, one sync). Frozen
        parameter caches (packed weights, folded BN) are rebuilt by the next (eager) run."""
        lib = L.lib()
        names = list(self.params) if names is None else list(names)
        total = sum(self.params[n].nbytes for n in names)
        pb = PinnedBuffer(max(total, 16))
        off = 0
        for name in names:
            arr = self.params[name]
            pb.u8[off:off + arr.nbytes] = np.ascontiguousarray(arr, np.float32).view(np.uint8).ravel()
            L.check(lib.sol_b200_plan_h2d(self.plan, self.buf[name], pb.ptr.value + off, arr.nbytes))
            off += arr.nbytes
        L.check(lib.sol_b200_plan_sync(self.plan))
        L.check(lib.sol_b200_plan_set_frozen(self.plan, 0))
        self._frozen = False
        self._ran = False

    def download_params(self, names=None) -> Dict[str, np.ndarray]:
        """Plan parameter buffers -> host arrays (one pinned staging area, one sync)."""
        lib = L.lib()
        names = list(self.params) if names is None else list(names)
        total = sum(self.params[n].nbytes for n in names)
        pb = PinnedBuffer(max(total, 16))
        offs, off = {}, 0
        for name in names:
            arr = self.params[name]
            L.check(lib.sol_b200_plan_d2h(self.plan, pb.ptr.value + off, self.buf[name], arr.nbytes))
            offs[name] = off
            off += arr.nbytes
        L.check(lib.sol_b200_plan_sync(self.plan))
        return {n: pb.u8[offs[n]:offs[n] + self.params[n].nbytes].view(np.float32).reshape(self.params[n].shape).copy()
                for n in names}

    def set_lr(self, lr: float) -> int:
        """Runtime learning rate of the plan's SgdUpdate steps (stream-ordered device write)."""
        n = C.c_int32()
        L.check(L.lib().sol_b200_plan_set_lr(self.plan, float(lr), C.byref(n)))
        self.lr = float(lr)
        return n.value

    # ------------------------------------------------------------------------------------------
    def load_state(self, params: Dict[str, np.ndarray]):
        """Replaces this plan's parameters; device caches are rebuilt."""
        for k, v in params.items():
            if k not in self.params or self.params[k].shape != np.shape(v):
                raise ValueError(f"parameter {k} mismatch")
            self.params[k] = np.asarray(v, np.float32).copy()
        self._upload_params(params.keys())

    def host_params(self) -> Dict[str, np.ndarray]:
        """This plan's device parameters, pulled back."""
        return self.download_params()

    def _validated(self, inputs: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
        out = {}
        for name, meta in self.inputs.items():
            if name not in inputs:
                raise KeyError(f"missing graph input '{name}'")
            a = np.asarray(inputs[name], np.float32)
            if a.size != meta.numel:
                raise ValueError(f"input '{name}' size mismatch")
            out[name] = a.reshape(meta.shape)
        return out

    def _wait_slot(self, k: int):
        """The pinned staging slot k is free once the copy that last read it has completed."""
        t = self._slot_ticket[k]
        if t is not None:
            L.check(L.lib().sol_b200_plan_copy_wait(self.plan, t))
            self._slot_ticket[k] = None

    def input_buffers(self) -> Dict[str, np.ndarray]:
        """Zero-copy serving: writable views of the free pinned staging slot (canonical NCHW f32).
        A data loader fills them in place, then stage_inputs() (no argument) ships them. Blocks only
        if the copy that last read this slot (two stages ago) is still running."""
        k = self._slot
        self._wait_slot(k)
        return {n: self.pin_in[n][k].view(np.float32, m.shape) for n, m in self.inputs.items()}

    def stage_inputs(self, inputs: Optional[Dict[str, np.ndarray]] = None):
        """Pipelined serving: (optionally fill the free pinned slot -- a parallel host copy --, then)
        start the host-to-device copy for the NEXT run() on the plan's copy stream. It overlaps the
        kernels of the run in flight; the next run() first moves the staged batch into the plan's
        input buffers. The two pinned slots alternate, and a slot is refilled only after the copy
        that read it completed (copy-stream fence), so staging batch i+1 never corrupts batch i."""
        lib = L.lib()
        k = self._slot
        self._wait_slot(k)
        if inputs is not None:
            arrs = self._validated(inputs)
            for name, meta in self.inputs.items():
                parallel_copy(self.pin_in[name][k].view(np.float32, meta.shape), arrs[name])
        for name, meta in self.inputs.items():
            L.check(lib.sol_b200_plan_stage_h2d(self.plan, self.in_canon[name], self.pin_in[name][k].ptr,
                                                4 * meta.numel))
        t = C.c_uint64()
        L.check(lib.sol_b200_plan_copy_fence(self.plan, C.byref(t)))
        self._slot_ticket[k] = t.value
        self._slot ^= 1

    def set_inputs(self, inputs: Dict[str, np.ndarray]):
        """Inputs of the next run() (host, canonical layout): staged through the pinned slots."""
        self.stage_inputs(inputs)

    def run(self):
        """One pass of the plan on its stream (no host synchronisation)."""
        lib = L.lib()
        use_graph = self.options.use_graph
        if not self._ran:
            # first run eagerly (module caches + kernel attributes), then freeze for inference
            L.check(lib.sol_b200_plan_run(self.plan, 0))
            self._ran = True
            if not self.options.train:
                L.check(lib.sol_b200_plan_set_frozen(self.plan, 1))
            if self.options.autotune and not self.tuned:
                autotune(self)
            return
        L.check(lib.sol_b200_plan_run(self.plan, int(use_graph)))

    def enqueue_fetch(self, names=None):
        """Device-to-host copies of outputs into the pinned output buffers, ordered on the plan
        stream after the runs already issued (no host synchronisation)."""
        lib = L.lib()
        names = list(self.graph.outputs) if names is None else names
        for n in names:
            meta = self.graph.meta_of(n)
            L.check(lib.sol_b200_plan_d2h(self.plan, self.pin_out[n].ptr, self.out_canon[n], 4 * meta.numel))

    def fetch_outputs(self, names=None) -> Dict[str, np.ndarray]:
        names = list(self.graph.outputs) if names is None else names
        self.enqueue_fetch(names)
        L.check(L.lib().sol_b200_plan_sync(self.plan))
        return {n: self.pin_out[n].view(np.float32, self.graph.meta_of(n).shape).copy() for n in names}

    def predict(self, inputs: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
        """fe::OptimizedModel::predict (frontend.hpp:119): host in, host out, canonical layouts."""
        self.set_inputs(inputs)
        self.run()
        return self.fetch_outputs()

    def train_step(self, batch: Dict[str, np.ndarray]) -> float:
        """fe::OptimizedModel::train_step(batch, lr, TrainMode::Native): forward, backward,
        gradient all-reduce (DP) and SGD on the device; returns the loss."""
        if not self.options.train:
            raise RuntimeError("model was not compiled for training")
        self.set_inputs(batch)
        self.run()
        return float(self.fetch_outputs([self.loss_name])[self.loss_name].reshape(()))

    def gradients(self) -> Dict[str, np.ndarray]:
        """Parameter gradients of the last step (canonical f32)."""
        lib = L.lib()
        out = {}
        for pname, gname in self.param_grads:
            shape = self.params[pname].shape
            pb = PinnedBuffer(4 * int(np.prod(shape)))
            L.check(lib.sol_b200_plan_d2h(self.plan, pb.ptr, self.buf[gname], 4 * int(np.prod(shape))))
            L.check(lib.sol_b200_plan_sync(self.plan))
            out[pname] = pb.view(np.float32, shape).copy()
        return out

    def read_tensor(self, name: str) -> np.ndarray:
        """Debug/parity access to any plan buffer still live (persistent or final values)."""
        lib = L.lib()
        meta = self.graph.meta_of(name) if name not in self.params else Meta("plain", self.params[name].shape)
        f32 = name in self.params or is_f32_tensor(self.graph, name)
        nbytes = storage_bytes(meta, self.dtype, f32)
        pb = PinnedBuffer(nbytes)
        L.check(lib.sol_b200_plan_d2h(self.plan, pb.ptr, self.buf[name], nbytes))
        L.check(lib.sol_b200_plan_sync(self.plan))
        return pb.u8[:nbytes].copy()

    # ------------------------------------------------------------------------------------------
    def profile(self) -> List[float]:
        """Per-step device times (us), CUDA events around every step (eager, no graph)."""
        lib = L.lib()
        n = C.c_int32()
        L.check(lib.sol_b200_plan_num_steps(self.plan, C.byref(n)))
        arr = (C.c_double * n.value)()
        L.check(lib.sol_b200_plan_profile(self.plan, arr, n.value))
        return list(arr)

    def event(self, slot: int):
        L.check(L.lib().sol_b200_plan_event_record(self.plan, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        L.check(L.lib().sol_b200_plan_event_elapsed(self.plan, a, b, C.byref(ms)))
        return ms.value

    def sync(self):
        L.check(L.lib().sol_b200_plan_sync(self.plan))

    def comm_info(self):
        """(nranks, rank, cuda device) of the plan's NCCL communicator, as NCCL reports them."""
        n, r, d = C.c_int32(), C.c_int32(), C.c_int32()
        L.check(L.lib().sol_b200_plan_comm_info(self.plan, C.byref(n), C.byref(r), C.byref(d)))
        return n.value, r.value, d.value

    def arena_bytes(self) -> int:
        v = C.c_uint64()
        L.check(L.lib().sol_b200_plan_arena_bytes(self.plan, C.byref(v)))
        return v.value

    def __del__(self):
        try:
            if getattr(self, "plan", None):
                L.lib().sol_b200_plan_destroy(self.plan)
                self.plan = None
        except Exception:
            pass


def activation_siblings(g: ModelGraph, units: List[ExecUnit]) -> Dict[str, tuple]:
    """DFP unit output -> (ReLU unit output, mask) where a single-op ReLU / ReLU6 unit reads the
    output of a straight-line BatchNorm [+ Add] unit (training graphs keep them apart because
    ReluBack needs the pre-activation tensor): one kernel writes both tensors."""
    by_out = {u.output: u for u in units}
    out = {}
    for u in units:
        if u.kind != "dfp" or len(u.node_ids) != 1:
            continue
        n = g.find_node(u.node_ids[0])
        if n.op not in ("ReLU", "ReLU6"):
            continue
        p = by_out.get(n.inputs[0])
        if p is None or p.kind != "dfp" or p.output in out:
            continue
        ops = [g.find_node(i).op for i in p.node_ids]
        if ops not in (["BatchNorm2d"], ["BatchNorm2d", "Add"]):
            continue
        out[p.output] = (u.output, 4 if n.op == "ReLU" else 8)
    return out


def bn_back_siblings(g: ModelGraph, units: List[ExecUnit]) -> Dict[str, tuple]:
    """BatchNormBackX unit output -> (BatchNormBackGamma output, BatchNormBackBeta output) of the
    same BatchNorm (same delta and x inputs); each sibling is a single-op unit."""
    single = {}
    for u in units:
        if len(u.node_ids) == 1:
            n = g.find_node(u.node_ids[0])
            if n.op in ("BatchNormBackX", "BatchNormBackGamma", "BatchNormBackBeta"):
                single[u.output] = n
    xs = {nm: n for nm, n in single.items() if n.op == "BatchNormBackX"}
    out = {}
    taken = set()
    for nm, nx in xs.items():
        gam = next((k for k, n in single.items() if n.op == "BatchNormBackGamma" and k not in taken
                    and list(n.inputs[:2]) == list(nx.inputs[:2])), None)
        # Beta reads only the delta, which two BatchNorms share behind an Add (residual block with
        # a downsample branch): assign one-to-one so every Beta tensor has exactly one writer
        bet = next((k for k, n in single.items() if n.op == "BatchNormBackBeta" and k not in taken
                    and n.inputs[0] == nx.inputs[0]), None)
        taken.update(k for k in (gam, bet) if k)
        if gam or bet:
            out[nm] = (gam, bet)
    return out


def gradient_completions(units: List[ExecUnit], siblings: Dict[str, tuple], absorbed) -> List[List[str]]:
    """Per unit of the plan (in order): the tensors its step completes -- its own output plus the
    BatchNormBackGamma/Beta siblings it writes; absorbed sibling units complete nothing."""
    out = []
    for u in units:
        if u.output in absorbed:
            out.append([])
        else:
            out.append([u.output] + [x for x in siblings.get(u.output, ()) if x])
    return out


# ------------------------------------------------------------------------------------------------
# autotune over B200 tile configurations (dnn::TuneCache / autotune, dnn.hpp:99-131, dnn.cpp:117-290)
# ------------------------------------------------------------------------------------------------

TUNE_VERSION = 1
TILE_CANDIDATES = {"conv": (0, 64, 65, 128, 256), "dual": (0, 128, 256)}


class TuneCache:
    """dnn::TuneCache (dnn.hpp:104-121): winners keyed by layer hyperparameters (never node ids),
    concurrent readers / exclusive writers, persisted as versioned JSON. A value is
    {"choice": {"tile_n": T}, "micros": t}."""

    def __init__(self):
        self._mu = threading.Lock()
        self._entries: Dict[str, dict] = {}

    @staticmethod
    def key(g: ModelGraph, unit: ExecUnit, dtype: int, device: str) -> str:
        parts = [device, f"dt{dtype}"]
        for nid in unit.node_ids:
            n = g.find_node(nid)
            a = n.attrs
            parts.append(f"{n.op}:{a.out_channels},{a.out_features},{a.kh},{a.kw},{a.sh},{a.sw},{a.ph},{a.pw},"
                         f"{a.groups},{int(a.has_bias)}")
        for nm in unit.inputs:
            parts.append("x" + "x".join(str(v) for v in g.meta_of(nm).shape))
        return "|".join(parts)

    def find(self, key: str) -> Optional[dict]:
        with self._mu:
            e = self._entries.get(key)
            return dict(e) if e else None

    def put(self, key: str, entry: dict):
        with self._mu:
            self._entries[key] = dict(entry)

    def size(self) -> int:
        with self._mu:
            return len(self._entries)

    def load(self, path: str):
        """A missing file leaves the cache empty; another format version is ignored."""
        try:
            with open(path) as f:
                d = json.load(f)
        except FileNotFoundError:
            return
        if d.get("version") != TUNE_VERSION:
            return
        with self._mu:
            self._entries.update(d.get("entries", {}))

    def save(self, path: str):
        with self._mu:
            d = {"version": TUNE_VERSION, "entries": dict(sorted(self._entries.items()))}
        tmp = path + ".tmp"
        with open(tmp, "w") as f:
            json.dump(d, f, indent=1)
        os.replace(tmp, path)


_TUNE_CACHE = TuneCache()


def _device_name(dev: int) -> str:
    try:
        import torch
        return torch.cuda.get_device_name(dev)
    except Exception:
        return "cuda"


def autotune(plan: "DevicePlan", cache: Optional[TuneCache] = None) -> Dict[int, dict]:
    """For every conv / linear forward step (and dual-GEMM tail) of a plan that has run once: time
    each B200 tile configuration (SOL_MODOPT_TILE_N) with the step alone on the plan's own buffers,
    keep the median of `tune_budget` runs, select the fastest, memoise it under the layer's
    hyperparameter key (dnn.cpp:214-290). Cache hits skip the measurement."""
    o = plan.options
    lib = L.lib()
    cache = cache or _TUNE_CACHE
    if o.tune_cache_path:
        cache.load(o.tune_cache_path)
    dev = _device_name(o.device)
    heavy_units = {u.output: u for u in plan.units if u.kind == "dnn"}
    out = {}
    for i, st in enumerate(plan.steps):
        if st.kind != "unit" or st.output not in heavy_units:
            continue
        u = heavy_units[st.output]
        fam = st.family
        if not (fam.startswith("conv_fprop") or fam.startswith("linear") or fam.startswith("conv_dgrad")):
            continue
        if fam.startswith("linear") and ("wgrad" in fam):
            continue
        cands = TILE_CANDIDATES["dual" if len(u.node_ids) >= 5 and fam == "conv_fprop_fused_tcgen05"
                                and sum(plan.graph.find_node(n).op == "Conv2d" for n in u.node_ids) == 2
                                else "conv"]
        key = TuneCache.key(plan.graph, u, plan.dtype, dev)
        hit = cache.find(key)
        if hit is not None:
            rc = lib.sol_b200_plan_step_set_option(plan.plan, i, L.MODOPT_TILE_N, int(hit["choice"]["tile_n"]))
            if rc == L.SOL_OK:
                plan.tune_cache_hits += 1
                out[i] = hit
                continue
        times = {}
        for t in cands:
            if lib.sol_b200_plan_step_set_option(plan.plan, i, L.MODOPT_TILE_N, t) != L.SOL_OK:
                continue
            us = C.c_double()
            L.check(lib.sol_b200_plan_time_step(plan.plan, i, max(1, o.tune_budget), C.byref(us)))
            plan.tuner_runs += max(1, o.tune_budget) + 1
            times[t] = us.value
        if not times:
            continue
        best = min(times, key=lambda t: (times[t], t != 0))  # ties keep the heuristic
        L.check(lib.sol_b200_plan_step_set_option(plan.plan, i, L.MODOPT_TILE_N, best))
        entry = {"choice": {"tile_n": best}, "micros": times[best], "candidates": {str(k): v for k, v in times.items()}}
        cache.put(key, entry)
        out[i] = entry
    if o.tune_cache_path:
        cache.save(o.tune_cache_path)
    plan.tuned = out or {"none": True}
    return out


# ------------------------------------------------------------------------------------------------
# the network API: fe::OptimizedModel (frontend.hpp:104-165)
# ------------------------------------------------------------------------------------------------

class TrainMode(enum.Enum):
    """fe::TrainMode (frontend.hpp:38)."""
    TRANSPARENT = 0  # forward + backward on the device, gradients round-trip, SGD on the host
    NATIVE = 1       # the whole step, SGD included, on the device


@dataclass
class CompileSummary:
    """fe::CompileSummary (frontend.hpp:63-69)."""
    units: int = 0
    dfp_units: int = 0
    dnn_units: int = 0
    kernels: int = 0
    reorders: int = 0
    tuner_runs: int = 0
    tune_cache_hits: int = 0
    compile_ms: float = 0.0
    cached: bool = False


class OptimizedModel:
    """fe::OptimizedModel over the B200 backend: a host master copy of the parameters, a forward
    plan and (for training models) a training plan, each with its parameter context -- the version
    of the host parameters its device buffers hold (ParamContext, frontend.hpp:137-145): a plan is
    re-uploaded only when the host parameters moved past it. After native training steps the
    training plan's device parameters are authoritative until sync_host_params() pulls them.

    Attribute access not defined here goes to the primary plan (the training plan of a training
    model, else the forward plan): run / stage_inputs / profile / steps / units / graph ..."""

    def __init__(self, g: ModelGraph, options: OptimizeOptions):
        t0 = time.perf_counter()
        self.__dict__["_plans"] = {}
        self.base = g
        self.options = options
        self.params: Dict[str, np.ndarray] = {k: np.asarray(v, np.float32).copy() for k, v in g.params.items()}
        self.param_version = 1
        self._ctx: Dict[bool, int] = {}         # plan (training?) -> parameter version it holds
        self._device_authoritative = False      # the training plan holds newer parameters
        self._mu = threading.RLock()
        self._primary = bool(options.train)
        self._plan(self._primary)
        self.summary = self._summarize((time.perf_counter() - t0) * 1e3)

    def __getattr__(self, name):
        plans = self.__dict__.get("_plans")
        if not plans:
            raise AttributeError(name)
        return getattr(plans[self.__dict__["_primary"]], name)

    # -- plans and parameter contexts ----------------------------------------------------------
    def _plan(self, training: bool) -> DevicePlan:
        if training not in self._plans:
            if training and not self.options.train:
                raise RuntimeError("model was not compiled for training")
            opts = dataclasses.replace(self.options, train=training)
            if not training:
                opts.world_size, opts.nccl_allreduce = 1, False
            p = DevicePlan(self.base if training else forward_graph(self.base), opts)
            self._plans[training] = p
            # a new plan holds the base graph's parameters: version 1 (ensure_context uploads newer)
            self._ctx[training] = 1
        return self._plans[training]

    def plan(self, training: bool = False) -> DevicePlan:
        """The device plan for inference or training (frontend.hpp:112), compiled on first use."""
        with self._mu:
            return self._plan(training)

    def _ensure_context(self, training: bool) -> DevicePlan:
        """ensure_context (frontend.hpp:145): the plan holds the current parameters."""
        p = self._plan(training)
        if self._device_authoritative and not training:
            self.sync_host_params()
        if self._ctx.get(training) != self.param_version:
            p.params = {k: v.copy() for k, v in self.params.items()}
            p._upload_params()
            self._ctx[training] = self.param_version
        return p

    # -- API ------------------------------------------------------------------------------------
    def load_state(self, params: Dict[str, np.ndarray]):
        """Replaces the host master parameters; every device context invalidates (frontend.hpp:115)."""
        with self._mu:
            for k, v in params.items():
                if k not in self.params or self.params[k].shape != np.shape(v):
                    raise ValueError(f"parameter {k} mismatch")
            for k, v in params.items():
                self.params[k] = np.asarray(v, np.float32).copy()
            self._device_authoritative = False
            self.param_version += 1
            self._ensure_context(self._primary)

    def predict(self, inputs: Dict[str, np.ndarray]) -> Dict[str, np.ndarray]:
        """Inference (frontend.hpp:119): host inputs in, canonical host outputs back. A training
        model runs its forward plan, synchronised with the latest trained parameters."""
        with self._mu:
            return self._ensure_context(False).predict(inputs)

    def train_step(self, batch: Dict[str, np.ndarray], lr: Optional[float] = None,
                   mode: TrainMode = TrainMode.NATIVE) -> float:
        """One SGD step, returns the loss (frontend.hpp:121-123). NATIVE: forward, backward,
        gradient all-reduce, SGD and the BN running statistics all on the device. TRANSPARENT:
        the device computes loss and gradients (its SGD runs with lr 0), the gradients come back
        and the host applies theta - lr * g in f32 (autodiff::sgd_step, autodiff.cpp:331-354)."""
        if not self.options.train:
            raise RuntimeError("model was not compiled for training")
        lr = self.options.lr if lr is None else float(lr)
        with self._mu:
            p = self._ensure_context(True)
            if mode == TrainMode.NATIVE:
                if p.lr != lr:
                    p.set_lr(lr)
                loss = p.train_step(batch)
                self.param_version += 1
                self._ctx[True] = self.param_version
                self._device_authoritative = True
                return loss
            if p.lr != 0.0:
                p.set_lr(0.0)
            loss = p.train_step(batch)
            grads = p.gradients()
            self._device_authoritative = True
            self.sync_host_params()  # running statistics (and the unchanged weights)
            lr32 = np.float32(lr)
            for name, gr in grads.items():
                self.params[name] = (self.params[name] - lr32 * gr.astype(np.float32)).astype(np.float32)
            self.param_version += 1
            p.params = {k: v.copy() for k, v in self.params.items()}
            p._upload_params(grads.keys())
            self._ctx[True] = self.param_version
            return loss

    def sync_host_params(self):
        """Pulls the device-resident parameters into the host master copy after native training
        (frontend.hpp:127); a no-op when the host copy is current."""
        with self._mu:
            if not self._device_authoritative:
                return
            got = self._plans[True].download_params()
            for k, v in got.items():
                self.params[k] = v
            self._plans[True].params = {k: v.copy() for k, v in got.items()}
            self._device_authoritative = False
            self._ctx[True] = self.param_version

    def host_params(self) -> Dict[str, np.ndarray]:
        """The host master parameters, synchronised first (frontend.hpp:128)."""
        with self._mu:
            self.sync_host_params()
            return {k: v.copy() for k, v in self.params.items()}

    def gradients(self) -> Dict[str, np.ndarray]:
        return self._plan(True).gradients()

    def export_bundle(self, directory: str, force: bool = False) -> str:
        """frontend.hpp:131: manifest + weights (SOLW) of a self-contained deployment bundle; returns
        the manifest path. run_bundle() replays it bit-identically to this model's predict()."""
        from .graph import model_to_json, weights_to_bytes
        man = os.path.join(directory, "manifest.json")
        if os.path.exists(man) and not force:
            raise FileExistsError(f"{man} exists (force=True overwrites)")
        os.makedirs(directory, exist_ok=True)
        with self._mu:
            self.sync_host_params()
            fwd = self._plan(False)
            params = {k: v.copy() for k, v in self.params.items()}
        g = forward_graph(self.base)
        g2 = ModelGraph(graph_inputs=g.graph_inputs, nodes=g.nodes, outputs=g.outputs, params=params)
        with open(os.path.join(directory, "weights.solw"), "wb") as f:
            f.write(weights_to_bytes(params))
        opts = {k: v for k, v in dataclasses.asdict(self.options).items()
                if k not in ("nccl_id", "world_size", "rank", "nccl_allreduce", "train", "device", "tune_cache_path",
                             "cache", "autotune")}
        manifest = {
            "format": "solb200-bundle", "version": 1,
            "library_sha256": library_sha256(),
            "model": json.loads(model_to_json(g2)),
            "weights": "weights.solw",
            "options": opts,
            "env": {k: v for k, v in os.environ.items() if k.startswith("SOL_")},
            "plan": {"units": [[u.kind, list(u.node_ids), u.output] for u in fwd.units],
                     "steps": [[st.kind, st.family, st.output] for st in fwd.steps],
                     "tiles": {str(k): v["choice"]["tile_n"] for k, v in fwd.tuned.items() if k != "none"}},
            "inputs": {n: list(m.shape) for n, m in fwd.inputs.items()},
            "outputs": list(fwd.graph.outputs),
        }
        with open(man, "w") as f:
            json.dump(manifest, f, indent=1)
        return man

    def _summarize(self, ms: float) -> CompileSummary:
        p = self._plans[self._primary]
        return CompileSummary(units=len(p.units), dfp_units=sum(u.kind == "dfp" for u in p.units),
                              dnn_units=sum(u.kind == "dnn" for u in p.units),
                              kernels=sum(st.launches for st in p.steps if st.kind != "allreduce"),
                              reorders=sum(st.kind == "reorder" for st in p.steps),
                              tuner_runs=p.tuner_runs, tune_cache_hits=p.tune_cache_hits, compile_ms=ms)


def forward_graph(g: ModelGraph) -> ModelGraph:
    """The inference graph of a training model: a CrossEntropyLoss output is replaced by its
    prediction input, and graph inputs only the loss read (the labels) are dropped."""
    losses = [n for n in g.nodes if n.op == "CrossEntropyLoss" and n.id in g.outputs]
    if not losses:
        return g
    drop = {n.id for n in losses}
    outs = []
    for o in g.outputs:
        if o in drop:
            p = g.find_node(o).inputs[0]
            if p not in outs:
                outs.append(p)
        elif o not in outs:
            outs.append(o)
    nodes = [n for n in g.nodes if n.id not in drop]
    used = {i for n in nodes for i in n.inputs} | set(outs)
    return ModelGraph([gi for gi in g.graph_inputs if gi.name in used], nodes, outs, g.params)


def library_sha256() -> str:
    h = hashlib.sha256()
    with open(L.LIB_PATH, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def run_bundle(directory: str, inputs: Dict[str, np.ndarray], device: int = 0,
               allow_other_library: bool = False) -> Dict[str, np.ndarray]:
    """fe::run_bundle (frontend.hpp:180): replays an exported bundle -- the same plan (verified
    unit by unit and step by step against the manifest) with the same kernels (library hash) and
    tile choices -- so the outputs are bit-identical to the exporting model's predict()."""
    from .graph import model_from_json
    with open(os.path.join(directory, "manifest.json")) as f:
        man = json.load(f)
    if man.get("format") != "solb200-bundle" or man.get("version") != 1:
        raise ValueError("not a solb200 bundle (format / version)")
    if man["library_sha256"] != library_sha256() and not allow_other_library:
        raise RuntimeError("bundle was exported with another libsolb200 build (bit-identity not guaranteed)")
    with open(os.path.join(directory, man["weights"]), "rb") as f:
        g = model_from_json(json.dumps(man["model"]), f.read())
    saved = {k: os.environ.get(k) for k in man.get("env", {})}
    os.environ.update(man.get("env", {}))
    try:
        kw = dict(man["options"], device=device, train=False, cache=False, autotune=False)
        opts = OptimizeOptions(**kw)
        m = optimize(g, opts)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    fwd = m.plan(False)
    units = [[u.kind, list(u.node_ids), u.output] for u in fwd.units]
    steps = [[st.kind, st.family, st.output] for st in fwd.steps]
    if units != man["plan"]["units"] or steps != man["plan"]["steps"]:
        raise RuntimeError("bundle plan mismatch: the rebuilt plan differs from the exported one")
    for k, t in man["plan"].get("tiles", {}).items():
        L.check(L.lib().sol_b200_plan_step_set_option(fwd.plan, int(k), L.MODOPT_TILE_N, int(t)))
    return m.predict(inputs)


# compiled-model cache: (graph structure, options) -> live model (fe::Engine model cache,
# frontend.hpp:93-94); weak, so a model no caller holds releases its device memory
_MODEL_CACHE: "weakref.WeakValueDictionary[str, OptimizedModel]" = weakref.WeakValueDictionary()
_CACHE_MU = threading.Lock()


def _structure_key(g: ModelGraph, options: OptimizeOptions) -> str:
    from .graph import model_to_json
    h = hashlib.sha256(model_to_json(g).encode())
    for k in sorted(g.params):
        h.update(k.encode())
        h.update(str(np.shape(g.params[k])).encode())
    h.update(options.fingerprint().encode())
    return h.hexdigest()


def optimize(g: ModelGraph, options: OptimizeOptions) -> OptimizedModel:
    """fe::optimize_graph (frontend.hpp:173-180): infer_shapes -> [build_training_graph] ->
    run_pipeline -> partition -> module compile -> plan. Results are cached on (structure,
    options): a repeated call returns the live cached model with `g`'s weights loaded
    (summary.cached = True)."""
    if not options.cache or options.world_size > 1:
        return OptimizedModel(g, options)
    key = _structure_key(g, options)
    with _CACHE_MU:
        m = _MODEL_CACHE.get(key)
    if m is not None:
        t0 = time.perf_counter()
        if any(not np.array_equal(m.params[k], v) for k, v in g.params.items()):
            m.load_state(g.params)
        m.summary = dataclasses.replace(m.summary, cached=True, compile_ms=(time.perf_counter() - t0) * 1e3)
        return m
    m = OptimizedModel(g, options)
    with _CACHE_MU:
        _MODEL_CACHE[key] = m
    return m


def nccl_unique_id() -> bytes:
    arr = (C.c_uint8 * 128)()
    L.check(L.lib().sol_b200_nccl_unique_id(arr))
    return bytes(arr)
