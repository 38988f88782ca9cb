"""Batch-sharded data parallelism host logic (paper_2003_10688_b200/dp.py) on CPU with gloo,
world_size 2: the same rank/shard/average/max protocol the NCCL plan runs on B200s.

The property checked end to end: for a model whose loss is a batch mean and whose layers have no
cross-sample coupling (no BatchNorm batch statistics), the average over ranks of each rank's
shard gradient equals the full-batch gradient (oracle, f64) -- i.e. the all-reduce(sum) x 1/G
step in the plan is exactly data-parallel SGD."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_10688_b200 import dp


def test_shard_covers_batch_exactly():
    x = np.arange(24).reshape(12, 2)
    parts = [dp.shard(x, r, 3) for r in range(3)]
    assert np.array_equal(np.concatenate(parts), x)
    with pytest.raises(ValueError):
        dp.shard(x, 0, 5)


def test_env_context_defaults(monkeypatch):
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    c = dp.env_context()
    assert (c.rank, c.world, c.local_rank) == (0, 1, 0)
    assert dp.max_over_ranks(3.5) == 3.5


def _bn_free_model():
    from paper_2003_10688_b200 import graph
    b = graph.GraphBuilder(11)
    b.input("x", graph.meta_nchw(0, 3, 8, 8))
    c = b.conv("c0", "x", 3, 8, 3, 1, 1)
    r = b.relu("r0", c)
    p = b.maxpool("p0", r, 2)
    f = b.flatten("flat", p)
    fc = b.linear("fc", f, 8 * 4 * 4, 5)
    prob = b.softmax("prob", fc)
    b.input("t", graph.meta_nc(0, 5))
    return b.done([b.ce("loss", prob, "t")])


def _grads(g, x, t):
    from oracle import sol_oracle as O
    from paper_2003_10688_b200 import autodiff, graph
    batch = x.shape[0]
    tg = autodiff.build_training_graph(graph.infer_shapes(g, batch))
    env = O.run_graph(graph.infer_shapes(tg.graph, batch), {"x": x, "t": t}, store_f32=False)
    return {p: np.asarray(env[gn], np.float64) for p, gn in tg.param_grads}


def _data(batch=8):
    rng = np.random.default_rng(4)
    x = rng.uniform(-1, 1, (batch, 3, 8, 8))
    t = np.zeros((batch, 5))
    t[np.arange(batch), rng.integers(0, 5, batch)] = 1
    return x, t


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = dp.env_context()
        assert (ctx.rank, ctx.world) == (rank, world)
        g = _bn_free_model()
        x, t = _data()
        local = _grads(g, dp.shard(x, rank, world), dp.shard(t, rank, world))
        avg = dp.average_gradients_host(local)
        slowest = dp.max_over_ranks(float(rank + 1))
        q.put((rank, {k: v.astype(np.float64) for k, v in avg.items()}, slowest))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dp_average_equals_full_batch_gradient_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _grads(_bn_free_model(), *_data())
    for rank, avg, slowest in results:
        assert slowest == float(world)
        assert sorted(avg) == sorted(full)
        for k in full:
            # gradients travel as f32 through the all-reduce
            np.testing.assert_allclose(avg[k], full[k], rtol=2e-5, atol=1e-6, err_msg=k)
    # every rank ends with the identical averaged gradient (replicas stay in lockstep)
    a, b = results[0][1], results[1][1]
    assert all(np.array_equal(a[k], b[k]) for k in a)
