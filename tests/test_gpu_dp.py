"""Two-rank NCCL data parallelism through the plan itself: each rank trains on its
shard with world_size=2; the plan all-reduces every gradient (ncclAvg, bucketed on the comm stream)
before the on-device SGD. The averaged shard gradients must equal the single-replica full-batch
gradient, both replicas must hold bit-identical gradients and parameters, and the plan's
communicator must span 2 ranks on 2 distinct GPUs. Needs >= 2 GPUs (skipped otherwise: gpurun
boxes have one GPU; the schedule itself is covered on CPU by tests/test_dp.py with gloo)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _model():
    from tests.test_dp import _bn_free_model
    return _bn_free_model()


def _data(batch=16):
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (batch, 3, 8, 8)).astype(np.float32)
    t = np.zeros((batch, 5), np.float32)
    t[np.arange(batch), rng.integers(0, 5, batch)] = 1
    return x, t


def _worker(rank, world, port, bucket_mb, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), SOL_AR_BUCKET_MB=bucket_mb)
    from paper_2003_10688_b200 import dp, frontend
    ctx = dp.init("nccl")
    try:
        x, t = _data()
        m = frontend.optimize(_model(), frontend.OptimizeOptions(
            batch=x.shape[0] // world, dtype="f32", train=True, lr=0.05, device=ctx.local_rank,
            world_size=world, rank=rank, nccl_id=ctx.nccl_id))
        loss = m.train_step({"x": dp.shard(x, rank, world), "t": dp.shard(t, rank, world)})
        q.put((rank, loss, m.gradients(), m.host_params(), m.comm_info(), m.ar_buckets))
    finally:
        import torch.distributed as dist
        dist.destroy_process_group()


@pytest.mark.skipif(_n_gpus() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("bucket_mb", ["25", "0.001"])
def test_two_rank_plan_allreduce_equals_full_batch(gpu, bucket_mb):
    import torch.multiprocessing as mp
    from paper_2003_10688_b200 import frontend
    world = 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, bucket_mb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    x, t = _data()
    full = frontend.optimize(_model(), frontend.OptimizeOptions(batch=x.shape[0], dtype="f32", train=True, lr=0.05))
    full_loss = full.train_step({"x": x, "t": t})
    fg = full.gradients()
    (r0, l0, g0, p0, c0, b0), (r1, l1, g1, p1, c1, b1) = res
    assert c0[0] == 2 and c1[0] == 2 and {c0[1], c1[1]} == {0, 1} and c0[2] != c1[2]
    if bucket_mb != "25":
        assert b0 > 1
    # the mean of the shard losses is the full-batch loss (CE is a batch mean)
    np.testing.assert_allclose((l0 + l1) / 2, full_loss, rtol=2e-3)
    for k in fg:
        assert np.array_equal(g0[k], g1[k]), k        # replicas hold the identical reduced gradient
        assert np.array_equal(p0[k], p1[k]), k        # ... and take the identical SGD step
        np.testing.assert_allclose(g0[k], fg[k], rtol=2e-3, atol=2e-4 * np.abs(fg[k]).max(), err_msg=k)
