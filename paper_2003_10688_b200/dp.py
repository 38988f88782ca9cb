"""Batch-sharded data parallelism (one process per GPU) — new relative to the reference, whose
SPEC lists distributed data parallelism as a non-goal.

Inference: each rank runs the full plan on its own shard of the global batch; no collective.
Training: each rank computes gradients of its shard (per-GPU BatchNorm statistics, DDP
semantics); the plan all-reduces every parameter gradient with NCCL over NVLink (sum, then x 1/G)
before the identical on-device SGD update on every replica. torch.distributed is only used to
bootstrap: rank 0's ncclUniqueId is broadcast, and bench timings are max-reduced over ranks.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np


@dataclass
class DPContext:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    nccl_id: Optional[bytes] = None


def env_context() -> DPContext:
    return DPContext(int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
                     int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str = "nccl") -> DPContext:
    """Initialise torch.distributed from the torchrun environment and share an NCCL id."""
    ctx = env_context()
    if ctx.world <= 1:
        return ctx
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        torch.cuda.set_device(ctx.local_rank)
    if not dist.is_initialized():
        dist.init_process_group(backend)
    obj = [None]
    if ctx.rank == 0:
        from .frontend import nccl_unique_id
        obj[0] = nccl_unique_id()
    dist.broadcast_object_list(obj, src=0)
    ctx.nccl_id = obj[0]
    return ctx


def shard(batch: np.ndarray, rank: int, world: int) -> np.ndarray:
    """Contiguous shard of a global batch along N (ranks get equal shards)."""
    n = batch.shape[0]
    if n % world:
        raise ValueError(f"global batch {n} not divisible by world size {world}")
    per = n // world
    return batch[rank * per:(rank + 1) * per]


def max_over_ranks(value: float) -> float:
    """Max of a host scalar over all ranks (timings are reported as the slowest rank)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_schedule(completions: List[List[str]], grad_bytes: Dict[str, float],
                       bucket_limit: float) -> Dict[int, List[str]]:
    """The training plan's gradient all-reduce buckets: walking the plan's units in
    order, each parameter gradient joins the pending bucket when the unit that completes it runs;
    the bucket is issued right after the unit that brings it to >= bucket_limit bytes, and the
    remainder after the last unit. Returns {unit index: [gradient names]} -- every gradient exactly
    once, never before its producer. The plan issues each bucket as one NCCL group on its comm
    stream (sum x 1/G = ncclAvg), overlapping the backward units that follow."""
    out: Dict[int, List[str]] = {}
    pending: List[str] = []
    size = 0.0
    seen = set()
    last = len(completions) - 1
    for i, names in enumerate(completions):
        for n in names:
            if n in grad_bytes and n not in seen:
                seen.add(n)
                pending.append(n)
                size += grad_bytes[n]
        if pending and (size >= bucket_limit or i == last):
            out[i] = pending
            pending, size = [], 0.0
    missing = set(grad_bytes) - seen
    if missing:
        raise ValueError(f"gradients never produced by a plan unit: {sorted(missing)[:4]}")
    return out
