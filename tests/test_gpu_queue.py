"""The device queue (sol_b200_queue_*, the rt::CommandQueue mirror) through the C ABI, ported from
the reference's own runtime tests (proj/tests/test_runtime.cpp):

* malloc preconditions, fresh-queue refs, the malloc/free lifecycle and every deferred error kind
  (:74-135): first error wins, later commands are skipped, repeated synchronize is idempotent;
* H2D snapshots the host range at enqueue time (runtime.hpp:106);
* byte counters are exact regardless of packing (:457-472) and >= 64 KiB runs of adjacent copies
  coalesce into ONE packed transfer (:136-195, here a real pinned DMA plus a scatter kernel);
* linearizability: 1000 random programs (malloc / free / copy in / copy out / ReLU launch / barrier)
  give byte-identical host results to a synchronous oracle, with and without coalescing (:437-455);
* B200 allocator properties: the pinned staging pool stops growing once warm (no cudaMallocHost in
  steady state), and a full device arena grows by a stream-ordered slab instead of failing.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OK, UAF, UNKNOWN, OOB = 0, 1, 2, 3


@pytest.fixture(scope="module")
def L():
    from paper_2003_10688_b200 import _lib
    return _lib


class Q:
    def __init__(self, L, coalesce=True, arena=64 << 20):
        self.L, self.lib = L, L.lib()
        self.h = C.c_void_p()
        L.check(self.lib.sol_b200_queue_create(0, arena, int(coalesce), C.byref(self.h)))
        self.keep = []

    def malloc(self, n):
        v = C.c_uint64()
        rc = self.lib.sol_b200_malloc_async(self.h, n, C.byref(v))
        if rc:
            raise self.L.SolError(rc, self.lib.sol_b200_last_error().decode())
        return v.value

    def free(self, v):
        return self.lib.sol_b200_free_async(self.h, v)

    def h2d(self, v, data: bytes):
        buf = C.create_string_buffer(data, len(data))
        self.L.check(self.lib.sol_b200_memcpy_h2d(self.h, v, buf, len(data)))
        return buf

    def d2h(self, v, n):
        buf = C.create_string_buffer(n)
        self.keep.append(buf)
        self.L.check(self.lib.sol_b200_memcpy_d2h(self.h, buf, v, n))
        return buf

    def launch(self, mod, args):
        arr = (C.c_uint64 * len(args))(*args)
        self.L.check(self.lib.sol_b200_launch(self.h, mod, arr, len(args)))

    def barrier(self):
        self.L.check(self.lib.sol_b200_barrier(self.h))

    def sync(self):
        msg = C.create_string_buffer(256)
        return self.lib.sol_b200_synchronize(self.h, msg, 256)

    def stats(self):
        s = self.L.TransferStats()
        self.L.check(self.lib.sol_b200_stats(self.h, C.byref(s)))
        return s

    def __del__(self):
        try:
            self.lib.sol_b200_queue_destroy(self.h)
        except Exception:
            pass


def add(L, v, d):
    out = C.c_uint64()
    L.check(L.lib().sol_b200_vptr_add(v, d, C.byref(out)))
    return out.value


_RELU = {}


def relu_module(n):
    """A one-op ReLU unit over [1, n] f32 (n % 4 == 0: no row padding): args = in, out."""
    if n not in _RELU:
        from paper_2003_10688_b200 import dfp, graph, partition
        b = graph.GraphBuilder(1)
        b.input("x", graph.meta_nc(0, n))
        g = graph.infer_shapes(b.done([b.relu("r", "x")]), 1)
        (u,) = partition.partition(g)
        _RELU[n] = dfp.create_module(g, u, 0)
    return _RELU[n].handle


def test_malloc_preconditions(gpu, L):
    q = Q(L)
    for bad in (0, 1 << 32):
        v = C.c_uint64()
        assert q.lib.sol_b200_malloc_async(q.h, bad, C.byref(v)) == L.SOL_E_INVALID_ARGUMENT


def test_fresh_queue_first_ref_is_one(gpu, L):
    q = Q(L)
    s = q.stats()
    assert s.h2d_bytes == 0 and s.launches == 0
    assert q.malloc(64) == 1 << 32
    assert q.sync() == OK
    assert Q(L).malloc(64) == 1 << 32  # refs are per queue


def test_clean_lifecycle_and_zeroed_malloc(gpu, L):
    q = Q(L)
    p = q.malloc(128)
    out = q.d2h(p, 128)
    q.free(p)
    assert q.sync() == OK
    assert out.raw == bytes(128)  # fresh allocations read as zeros (reference: vector resize)


def test_launch_after_free_is_use_after_free(gpu, L):
    q = Q(L)
    a, b = q.malloc(32), q.malloc(32)
    q.free(a)
    q.launch(relu_module(8), [a, b])
    assert q.sync() == UAF
    assert q.sync() == UAF  # repeated synchronize is idempotent


def test_double_free_is_unknown_ref(gpu, L):
    q = Q(L)
    p = q.malloc(16)
    q.free(p)
    assert q.free(p) == OK  # deferred, not eager
    assert q.sync() == UNKNOWN


def test_offset_free_rejected_eagerly(gpu, L):
    q = Q(L)
    p = q.malloc(16)
    assert q.free(add(L, p, 4)) == L.SOL_E_INVALID_ARGUMENT
    assert q.sync() == OK


def test_out_of_bounds_copy_surfaces_at_synchronize(gpu, L):
    q = Q(L)
    p = q.malloc(16)
    q.h2d(add(L, p, 8), bytes(16))  # 8 + 16 > 16
    assert q.sync() == OOB


def test_first_error_wins_and_later_commands_are_skipped(gpu, L):
    q = Q(L)
    a = q.malloc(64)
    q.free(a)
    q.h2d(a, bytes(64))                 # use after free (first)
    b = q.malloc(16)
    q.h2d(add(L, b, 8), bytes(16))      # out of bounds (skipped: the first error wins)
    assert q.sync() == UAF


def test_h2d_snapshots_at_enqueue(gpu, L):
    q = Q(L)
    p = q.malloc(4096)
    host = C.create_string_buffer(b"\x01" * 4096, 4096)
    L.check(q.lib.sol_b200_memcpy_h2d(q.h, p, host, 4096))
    C.memset(host, 2, 4096)  # mutate after enqueue, before the copy can have run
    out = q.d2h(p, 4096)
    assert q.sync() == OK
    assert out.raw == b"\x01" * 4096


@pytest.mark.parametrize("coalesce", [True, False])
def test_byte_counters_exact_regardless_of_packing(gpu, L, coalesce):
    q = Q(L, coalesce)
    rng = np.random.default_rng(9)
    p = q.malloc(1 << 20)
    want = 0
    for _ in range(50):
        n = int(4 * (1 + rng.integers(0, 1024)))
        q.h2d(p, bytes(n))
        want += n
    q.d2h(p, 4096)
    assert q.sync() == OK
    s = q.stats()
    assert (s.h2d_bytes, s.h2d_ops, s.d2h_bytes, s.d2h_ops) == (want, 50, 4096, 1)


@pytest.mark.parametrize("coalesce", [True, False])
def test_copy_runs_coalesce_into_one_packed_transfer(gpu, L, coalesce):
    q = Q(L, coalesce)
    p = q.malloc(102400)
    chunks = [bytes([i % 251]) * 1024 for i in range(100)]
    for i, c in enumerate(chunks):
        q.h2d(add(L, p, 1024 * i), c)
    out = q.d2h(p, 102400)
    assert q.sync() == OK
    assert out.raw == b"".join(chunks)
    assert q.stats().packed_transfers == (1 if coalesce else 0)


def _random_program(rng):
    """proj/tests/test_runtime.cpp:275-343: valid programs over numbered slots."""
    steps, sizes, alive, hostbufs = [], [], [], 0
    for _ in range(int(rng.integers(1, 40))):
        op = int(rng.integers(0, 6))
        if op == 0:
            sizes.append(int(16 * (1 + rng.integers(0, 64))))
            alive.append(True)
            steps.append(("malloc", len(sizes) - 1))
        elif op == 1 and sizes:
            i = int(rng.integers(0, len(sizes)))
            if alive[i]:
                alive[i] = False
                steps.append(("free", i))
        elif op in (2, 3) and sizes:
            i = int(rng.integers(0, len(sizes)))
            if alive[i]:
                n = 4 * int(1 + rng.integers(0, sizes[i] // 4))
                off = 4 * int(rng.integers(0, (sizes[i] - n) // 4 + 1))
                if op == 2:
                    steps.append(("in", i, off, rng.integers(0, 256, n, dtype=np.uint8).tobytes()))
                else:
                    steps.append(("out", i, off, n, hostbufs))
                    hostbufs += 1
        elif op == 4 and len(sizes) >= 2:
            a, b = (int(v) for v in rng.integers(0, len(sizes), 2))
            if alive[a] and alive[b] and a != b:
                steps.append(("relu", a, b, min(sizes[a], sizes[b]) // 4))
        elif op == 5:
            steps.append(("barrier",))
    return steps, sizes, hostbufs


def _oracle(steps, sizes, nhost):
    mem, out = {}, [b""] * nhost
    for s in steps:
        if s[0] == "malloc":
            mem[s[1]] = bytearray(sizes[s[1]])
        elif s[0] == "free":
            del mem[s[1]]
        elif s[0] == "in":
            mem[s[1]][s[2]:s[2] + len(s[3])] = s[3]
        elif s[0] == "out":
            out[s[4]] = bytes(mem[s[1]][s[2]:s[2] + s[3]])
        elif s[0] == "relu":
            x = np.frombuffer(bytes(mem[s[1]][:4 * s[3]]), np.float32)
            y = np.where(x > 0, x, np.float32(0)).astype(np.float32)  # NaN -> 0 like `x > 0 ? x : 0`
            mem[s[2]][:4 * s[3]] = y.tobytes()
    return out


def _run_async(q, steps, sizes, nhost, L):
    ptrs, bufs, keep = {}, {}, []
    for s in steps:
        if s[0] == "malloc":
            ptrs[s[1]] = q.malloc(sizes[s[1]])
        elif s[0] == "free":
            q.free(ptrs[s[1]])
        elif s[0] == "in":
            keep.append(q.h2d(add(L, ptrs[s[1]], s[2]), s[3]))
        elif s[0] == "out":
            bufs[s[4]] = q.d2h(add(L, ptrs[s[1]], s[2]), s[3])
        elif s[0] == "relu":
            q.launch(relu_module(s[3]), [ptrs[s[1]], ptrs[s[2]]])
        elif s[0] == "barrier":
            q.barrier()
    assert q.sync() == OK
    return [bufs[i].raw for i in range(nhost)]


def test_linearizability_1000_random_programs(gpu, L):
    rng = np.random.default_rng(2024)
    qs = {True: Q(L, True), False: Q(L, False)}
    for trial in range(1000):
        steps, sizes, nhost = _random_program(rng)
        # the ReLU module's arguments are [1, n] f32 with n % 4 == 0 (no row padding)
        steps = [s if s[0] != "relu" else (s[0], s[1], s[2], s[3] // 4 * 4) for s in steps]
        steps = [s for s in steps if not (s[0] == "relu" and s[3] == 0)]
        want = _oracle(steps, sizes, nhost)
        for co, q in qs.items():
            got = _run_async(q, steps, sizes, nhost, L)
            assert got == want, (trial, co)
    for q in qs.values():
        assert q.stats().launches > 100


def test_pinned_pool_and_arena_growth(gpu, L):
    q = Q(L, True, arena=1 << 20)
    big = q.malloc(8 << 20)            # larger than the whole arena: a new stream-ordered slab
    assert q.stats().device_slabs == 2
    payload = bytes(range(256)) * (8 << 12)
    q.h2d(big, payload)
    out = q.d2h(big, len(payload))
    assert q.sync() == OK and out.raw == payload
    slabs = q.stats().pinned_slabs
    for _ in range(20):                # steady state: the staging pool is recycled
        q.h2d(big, payload)
        q.d2h(big, 4096)
        assert q.sync() == OK
    assert q.stats().pinned_slabs == slabs
