"""Batch-sharded data parallelism host logic (paper_2003_10688_b200/dp.py) on CPU with gloo,
world_size 2: the same rank/shard/bucket-schedule/average/max protocol the NCCL plan runs on
B200s. The training plan's own all-reduce schedule (dp.allreduce_schedule over the plan's units,
as frontend.OptimizedModel issues it) is executed unit by unit with the oracle and gloo.

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


def _plan_units(g, batch):
    """The training plan's unit list, sibling map and all-reduce bucket schedule, exactly as
    frontend.OptimizedModel builds them (pure host logic: no device needed)."""
    from paper_2003_10688_b200 import autodiff, frontend, graph, partition, passes
    tg = autodiff.build_training_graph(graph.infer_shapes(g, batch))
    cg = passes.run_pipeline(graph.infer_shapes(tg.graph, batch))
    units = partition.partition(cg)
    sib = frontend.bn_back_siblings(cg, units)
    absorbed = {v for pair in sib.values() for v in pair if v is not None}
    sched = dp.allreduce_schedule(frontend.gradient_completions(units, sib, absorbed),
                                  {gn: 4.0 * g.params[p].size for p, gn in tg.param_grads}, 512.0)
    return tg, cg, units, sib, absorbed, sched


def _simulate_plan(g, x, t, world):
    """Runs the training plan's units in plan order with the oracle (f64 math, f32 storage) on this
    rank's shard and issues the plan's all-reduce buckets (sum, then x 1/G in f32: ncclAvg) over
    the process group at the positions the plan issues them. Raises if a bucket would reduce a
    gradient before the unit producing it ran, or if a unit wrote a gradient after its reduction."""
    import torch
    import torch.distributed as dist
    from oracle import sol_oracle as O
    batch = x.shape[0]
    tg, cg, units, sib, absorbed, sched = _plan_units(g, batch)
    env = {"x": np.asarray(x, np.float32), "t": np.asarray(t, np.float32)}
    params = {k: np.asarray(v, np.float64) for k, v in g.params.items()}
    by_out = {u.output: u for u in units}
    reduced = {}

    def eval_unit(u):
        for nid in u.node_ids:
            n = cg.find_node(nid)
            assert nid not in reduced, f"{nid} written after its all-reduce"
            env[nid] = np.asarray(O.eval_node(n, [env[i] for i in n.inputs], params), np.float32)

    for ui, u in enumerate(units):
        if u.output not in absorbed:
            eval_unit(u)
            for s in sib.get(u.output, ()):  # the BatchNormBackX step also writes its siblings
                if s is not None:
                    eval_unit(by_out[s])
        for gname in sched.get(ui, ()):
            assert gname in env, f"bucket after unit {ui} reduces {gname} before it is computed"
            assert gname not in reduced, f"{gname} reduced twice"
            buf = torch.from_numpy(np.ascontiguousarray(env[gname], np.float32)).clone()
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)
            env[gname] = (buf * np.float32(1.0 / world)).numpy()
            reduced[gname] = env[gname].copy()
    assert sorted(reduced) == sorted(gn for _, gn in tg.param_grads)
    for gname, v in reduced.items():  # nothing touched a gradient after its bucket
        assert np.array_equal(env[gname], v), gname
    return {p: np.asarray(env[gn], np.float64) for p, gn in tg.param_grads}, len(sched)


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
        avg, buckets = _simulate_plan(g, dp.shard(x, rank, world), dp.shard(t, rank, world), world)
        slowest = dp.max_over_ranks(float(rank + 1))
        # a BatchNorm model (per-GPU batch statistics, BN-backward sibling outputs): the schedule
        # still reduces every gradient exactly once after its producer, and replicas agree
        from paper_2003_10688_b200 import models
        gr = models.resnet(18, hw=16, classes=5, width=8, train=True)
        xr = np.random.default_rng(5).uniform(-1, 1, (4, 3, 16, 16))
        tr = np.zeros((4, 5))
        tr[np.arange(4), np.arange(4) % 5] = 1
        avg_bn, buckets_bn = _simulate_plan(gr, dp.shard(xr, rank, world), dp.shard(tr, rank, world), world)
        q.put((rank, {k: v.astype(np.float64) for k, v in avg.items()}, slowest, buckets,
               {k: v for k, v in avg_bn.items()}, buckets_bn))
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
    for rank, avg, slowest, buckets, avg_bn, buckets_bn in results:
        assert slowest == float(world)
        assert buckets > 1 and buckets_bn > 1  # the 512-byte bucket limit forces several buckets
        assert sorted(avg) == sorted(full)
        for k in full:
            # gradients travel as f32 through the all-reduce
            np.testing.assert_allclose(avg[k], full[k], rtol=2e-5, atol=1e-6, err_msg=k)
    # every rank ends with the identical averaged gradients (replicas stay in lockstep)
    for i in (1, 4):
        a, b = results[0][i], results[1][i]
        assert all(np.array_equal(a[k], b[k]) for k in a)


def test_allreduce_schedule_buckets():
    comp = [["a"], [], ["b", "c"], ["x"], ["d"]]
    sizes = {"a": 10.0, "b": 10.0, "c": 30.0, "d": 5.0}
    assert dp.allreduce_schedule(comp, sizes, 25.0) == {2: ["a", "b", "c"], 4: ["d"]}
    assert dp.allreduce_schedule(comp, sizes, 1e9) == {4: ["a", "b", "c", "d"]}
    assert dp.allreduce_schedule(comp, sizes, 1.0) == {0: ["a"], 2: ["b", "c"], 4: ["d"]}
    with pytest.raises(ValueError):
        dp.allreduce_schedule(comp, dict(sizes, e=1.0), 1.0)
