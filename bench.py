#!/usr/bin/env python3
"""Benchmark: ResNet-50 bf16 inference, batch 256 per GPU (BASELINE.json configs[2]), batch-sharded
over N GPUs (one process per GPU, weak scaling), plus a ResNet-50 bf16 training step at batch 128
per GPU with NCCL gradient all-reduce (configs[3]) reported alongside.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--no-train]

Prints ONE JSON line on rank 0. `value` = whole-job images/s with inputs resident in HBM (CUDA
events on the plan stream, max over ranks); `e2e` = the same through the public API per step
(pinned-host H2D of the input batch, plan run, D2H of the probabilities). Synthetic data
(U(-1,1) images, random-init weights; no network for datasets/checkpoints). Every step's working
set (154 MB input + ~4 GB activations) exceeds the 126 MB L2, so no explicit flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "images/sec ResNet-50 infer+train at 1/2/4/8 B200; % of HBM/TC roofline"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["active", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names[1:], parts[5:9]):
                if v.lower() in ("active", "0x1", "1"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_local_cpus(device: int):
    """Host cores on the GPU's NUMA node (pinned staging buffers allocated from these threads
    land in local memory, which keeps host-to-device bandwidth at the PCIe link rate)."""
    try:
        bus = subprocess.run(["nvidia-smi", "-i", str(device), "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                             capture_output=True, text=True, timeout=20).stdout.strip()
        dom, rest = bus.split(":", 1)
        path = f"/sys/bus/pci/devices/{dom[-4:].lower()}:{rest.lower()}/local_cpulist"
        cpus = set()
        for part in open(path).read().strip().split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part:
                cpus.add(int(part))
        return cpus & os.sched_getaffinity(0) or None
    except Exception:
        return None


# ------------------------------------------------------------------------------------------------
# reference CPU implementation (oracle/_ref: the reference's own compiled f32 path)
# ------------------------------------------------------------------------------------------------

def reference_throughput(model: str, hw: int, images: int, threads: int, classes: int = 1000):
    """Times the reference's compiled SOL CPU path (run_pipeline -> partition -> lower_group /
    run_kernel for DFP units + heuristic_choice / execute_choice for heavy layers, all from the
    unmodified reference sources built into oracle/_ref) on `images` single-image sessions spread
    over `threads` host threads (eval-mode BN makes images independent). Falls back to the numpy
    oracle port when the reference library is unavailable."""
    from paper_2003_10688_b200 import graph, models
    from oracle import refbridge
    g = models.resnet(50, hw=hw, classes=classes) if model == "resnet50" else models.resnet(18, hw=hw, classes=classes)
    rng = np.random.default_rng(0)
    xs = [rng.uniform(-1, 1, (1, 3, hw, hw)).astype(np.float32) for _ in range(images)]
    if refbridge.available():
        mj, wb = graph.model_to_json(g), graph.weights_to_bytes(g.params)
        sessions = []
        for _ in range(threads):
            s = refbridge.RefSession(mj, wb, 1)
            s.pipeline()
            sessions.append(s)
        todo = list(range(images))
        lock = threading.Lock()

        def worker(s):
            while True:
                with lock:
                    if not todo:
                        return
                    i = todo.pop()
                s.set_input("x", xs[i])
                s.run_compiled()

        t0 = time.perf_counter()
        ths = [threading.Thread(target=worker, args=(s,)) for s in sessions]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        dt = time.perf_counter() - t0
        return images / dt, "reference", dt
    from oracle import sol_oracle as O
    gi = graph.infer_shapes(g, 1)
    t0 = time.perf_counter()
    for x in xs:
        O.run_graph(gi, {"x": x})
    dt = time.perf_counter() - t0
    return images / dt, "port", dt


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    images = threads  # one image per host thread per step (bounded sample: ~8-10 s per step)
    vals = []
    kind = "reference"
    for i in range(args.warmup + args.steps):
        v, kind, dt = reference_throughput("resnet50", 224, images, threads)
        if i >= args.warmup:
            vals.append(v)
    value = float(np.mean(vals)) if vals else 0.0
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * images / value if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "ResNet-50 inference 224x224, reference compiled f32 CPU path (oracle/_ref)",
                   "model": "resnet50", "global_batch": images, "seq_len": 0,
                   "parallelism": f"{threads} host threads, one image per thread"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": kind,
                         "sample": f"{images} images of 3x224x224 per step"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# B200 arm
# ------------------------------------------------------------------------------------------------

def conv_traffic_profile(key):
    """ncu DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the dominant conv
    kernel, from the committed capture for THIS workload (profiles/conv_traffic_latest.json holds
    one entry per workload key); None when no capture exists for it."""
    try:
        with open(os.path.join(ROOT, "profiles", "conv_traffic_latest.json")) as f:
            tj = json.load(f)
    except Exception:
        return None
    e = tj.get(key) if isinstance(tj.get(key), dict) else (tj if tj.get("workload") == key else None)
    return e.get("mean_dram_bytes_per_launch") if e else None


def roofline_of(m, peaks, peaks_kind, families, bound, traffic=None):
    """Achieved throughput of one kernel family measured live with CUDA events around every plan
    step (one eager profiled pass): algorithmic FLOPs (or bytes) per launch / launch time."""
    times = m.profile()
    info = m.steps
    tot_t, tot_w = 0.0, 0.0
    for st, t in zip(info, times):
        if st.family in families:
            tot_t += t
            tot_w += st.algo_flops if bound == "tensor" else st.algo_bytes
    if tot_t <= 0:
        return None, times
    # speed of light per launch: max(FLOPs / tensor peak, bytes / HBM peak) -- many convolutions of
    # the network are HBM-bound, so this is the fraction that can actually approach 1
    tc_peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * 1e12
    hbm_peak = peaks["hbm_gbs"] * 1e9
    sol_t = sum(max(st.algo_flops / tc_peak, st.algo_bytes / hbm_peak) for st, t in zip(info, times)
                if st.family in families)
    if bound == "tensor":
        achieved = tot_w / (tot_t * 1e-6) / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        unit = "TFLOP/s"
    else:
        achieved = tot_w / (tot_t * 1e-6) / 1e9
        peak = peaks["hbm_gbs"]
        unit = "GB/s"
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
            "traffic": traffic, "kernel": "+".join(sorted(families)), "peak_source": peaks_kind,
            "share_of_step": tot_t / sum(times), "sol_frac": sol_t / (tot_t * 1e-6)}, times


def measured_launches(m):
    """Kernels of OURS (names in namespace solb200) one step launches, counted by CUPTI through
    torch.profiler over two untimed steps (graph-launched kernels included); None if profiling is
    unavailable (e.g. under ncu), in which case the plan's own per-unit count is reported."""
    if os.environ.get("SOL_BENCH_NO_LAUNCH_COUNT"):
        return None
    try:
        import warnings
        import torch
        warnings.filterwarnings("ignore", message="Warning: Profiler clears events")
        m.sync()
        with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
            for _ in range(2):
                m.run()
            m.sync()
            torch.cuda.synchronize()
        n = sum(1 for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and "solb200" in e.name)
        return n // 2 if n > 0 else None
    except Exception:
        return None


def bench_model(m, inputs, steps, warmup, out_names):
    """Device-timed steps (inputs resident) and end-to-end steps (H2D + run + D2H)."""
    from paper_2003_10688_b200 import dp
    m.set_inputs(inputs)
    for _ in range(max(warmup, 3)):
        m.run()
    m.sync()
    dp_barrier()
    m.event(0)
    for _ in range(steps):
        m.run()
    m.event(1)
    m.sync()
    dev_ms = m.elapsed_ms(0, 1) / steps
    dev_ms = dp.max_over_ranks(dev_ms)
    # end-to-end through the public API: every step copies its batch from pinned host memory to the
    # device and reads its result back; the input copy of step i+1 is staged on the plan's copy
    # stream while step i computes (OptimizedModel.stage_inputs). The pinned slots are filled in
    # place through OptimizedModel.input_buffers() -- what a data loader writing pinned memory does
    h2d = sum(4 * a.size for a in inputs.values())
    d2h = sum(4 * m.graph.meta_of(n).numel for n in out_names)

    def pipelined(k, fill):
        if fill:
            for name, v in m.input_buffers().items():
                v[...] = inputs[name]
        m.stage_inputs()
        for i in range(k):
            m.run()
            if i + 1 < k:
                if fill:
                    for name, v in m.input_buffers().items():
                        v[...] = inputs[name]
                m.stage_inputs()
            m.enqueue_fetch(out_names)

    pipelined(max(warmup, 3), True)  # warm-up: fills both pinned slots, primes the copy stream
    dp_barrier()
    m.sync()
    m.event(2)
    pipelined(steps, False)
    m.event(3)
    m.sync()
    e2e_ms = dp.max_over_ranks(m.elapsed_ms(2, 3) / steps)
    # the synchronous predict()/train_step() call from numpy arrays: the host copy into pinned
    # memory, H2D, the plan, D2H and the host synchronisation all on the critical path (wall clock)
    import time as _t
    k = min(steps, 10)
    call = (lambda: m.predict(inputs)) if m.loss_name is None else (lambda: m.train_step(inputs))
    call()
    dp_barrier()
    t0 = _t.perf_counter()
    for _ in range(k):
        call()
    sync_ms = dp.max_over_ranks((_t.perf_counter() - t0) * 1e3 / k)
    return dev_ms, e2e_ms, h2d, d2h, sync_ms


_DIST = False


def distinct_gpus(device: int) -> int:
    """Number of distinct physical GPUs (by UUID) the ranks of this job run on."""
    import torch
    uuid = str(torch.cuda.get_device_properties(device).uuid)
    if not _DIST:
        return 1
    import torch.distributed as dist
    got = [None] * dist.get_world_size()
    dist.all_gather_object(got, uuid)
    return len(set(got))


def comm_of(m, world: int):
    """The training plan's NCCL communicator as NCCL reports it (ncclCommCount / ncclCommCuDevice)."""
    if world == 1:
        return {"nranks": 1, "nranks_ok": True, "note": "single replica: no communicator"}
    n, r, d = m.comm_info()
    return {"nranks": n, "rank": r, "cuda_device": d, "nranks_ok": n == world}


def dp_barrier():
    if _DIST:
        import torch.distributed as dist
        dist.barrier()


def run_b200(args):
    global _DIST
    from paper_2003_10688_b200 import dp, frontend, models
    ctx = dp.init("nccl") if args.gpus > 1 else dp.env_context()
    _DIST = ctx.world > 1
    if ctx.world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but the process group has {ctx.world} ranks")
    device = ctx.local_rank
    all_cpus = os.sched_getaffinity(0)
    local = gpu_local_cpus(device)
    if local:
        os.sched_setaffinity(0, local)
    peaks, peaks_kind = load_peaks()
    B = args.batch
    rng = np.random.default_rng(1234 + ctx.rank)
    x = rng.uniform(-1, 1, (B, 3, 224, 224)).astype(np.float32)

    g = models.resnet(50, hw=224, classes=1000)
    m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype="bf16", device=device, fuse_epilogue=True))
    sampler = ClockSampler(device) if ctx.rank == 0 and not os.environ.get("SOL_BENCH_NO_CLOCKS") else None
    if sampler:
        sampler.start()
    dev_ms, e2e_ms, h2d, d2h, sync_ms = bench_model(m, {"x": x}, args.steps, args.warmup, ["prob"])
    clocks = sampler.stop() if sampler else None
    launches_per_step = measured_launches(m)
    if launches_per_step is None:
        launches_per_step = sum(s.launches_frozen for s in m.steps)  # the inference plan runs frozen
    world = ctx.world
    gpus_active = distinct_gpus(device)
    value = world * B / (dev_ms / 1e3)
    e2e = world * B / (e2e_ms / 1e3)
    conv_fams = {"conv_fprop_tcgen05", "conv_fprop_fused_tcgen05", "conv_stem_tcgen05", "conv_stem_fused_tcgen05"}
    roof, times = roofline_of(m, peaks, peaks_kind, conv_fams, "tensor",
                              traffic=conv_traffic_profile("resnet50_infer_b256_bf16"))
    dfp_fams = {s.family for s in m.steps if s.family.startswith("dfp_")}
    roof_dfp, _ = roofline_of(m, peaks, peaks_kind, dfp_fams, "hbm",
                              traffic=conv_traffic_profile("resnet50_infer_b256_bf16_dfp"))
    fam_time = {}
    for st, t in zip(m.steps, times):
        fam_time[st.family] = fam_time.get(st.family, 0.0) + t
    train = None
    if args.train:
        Bt = args.train_batch
        gt = models.resnet(50, hw=224, classes=1000, train=True)
        # autotune: the tcgen05 tile of every forward / data-gradient conv measured on the plan's own
        # buffers (frontend.autotune; ~1.5 s at start-up, ~1.5% faster steps)
        mt = frontend.optimize(gt, frontend.OptimizeOptions(batch=Bt, dtype="bf16", train=True, lr=0.01,
                                                            device=device, world_size=world, rank=ctx.rank,
                                                            nccl_id=ctx.nccl_id, autotune=True, tune_budget=3))
        t = np.zeros((Bt, 1000), np.float32)
        t[np.arange(Bt), rng.integers(0, 1000, Bt)] = 1
        xt = x[:Bt] if Bt <= B else rng.uniform(-1, 1, (Bt, 3, 224, 224)).astype(np.float32)
        tdev, te2e, th2d, td2h, tsync = bench_model(mt, {"x": xt, "t": t}, args.train_steps, args.warmup, ["loss"])
        troof, ttimes = roofline_of(mt, peaks, peaks_kind,
                                    {"conv_fprop_tcgen05", "conv_fprop_bnstats_tcgen05", "conv_dgrad_tcgen05", "conv_dgrad_fused_tcgen05",
                                     "conv_wgrad_tcgen05",
                                     "conv_stem_tcgen05", "conv_stem_wgrad_tcgen05"}, "tensor",
                                    traffic=conv_traffic_profile("resnet50_train_b128_bf16"))
        tfam = {}
        for st, tt in zip(mt.steps, ttimes):
            tfam[st.family] = tfam.get(st.family, 0.0) + tt
        train = {"metric": "images/sec ResNet-50 bf16 training (fwd+bwd+allreduce+SGD)",
                 "value": world * Bt / (tdev / 1e3), "unit": "images/s", "ms_per_step": tdev,
                 "global_batch": world * Bt, "per_gpu_batch": Bt,
                 "e2e": {"value": world * Bt / (te2e / 1e3), "unit": "images/s", "h2d_bytes_per_step": th2d,
                         "d2h_bytes_per_step": td2h, "source": "pinned host slots, H2D pipelined on the copy stream"},
                 "e2e_sync_call": {"value": world * Bt / (tsync / 1e3), "unit": "images/s",
                                   "api": "train_step(numpy batch) per step, wall clock"},
                 "comm": comm_of(mt, world),
                 "roofline": troof,
                 "autotuned_steps": len([k for k in mt.tuned if k != "none"]),
                 "gpu_launches": (measured_launches(mt) or sum(s.launches for s in mt.steps)) * args.train_steps,
                 "family_ms_per_step": {k: round(v / 1e3, 3) for k, v in sorted(tfam.items(), key=lambda kv: -kv[1])[:8]}}
    if ctx.rank != 0:
        return
    others = other_configs(args, peaks, peaks_kind, device) if (world == 1 and args.configs) else None
    os.sched_setaffinity(0, all_cpus)  # the CPU baseline uses every host core
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, kind, dt = reference_throughput("resnet50", 224, threads, threads)
        cpu = {"value": v, "unit": "images/s", "cores": threads, "kind": kind,
               "sample": f"{threads} images 3x224x224, one per host thread, {dt:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "ResNet-50 inference 224x224 bf16 (BASELINE configs[2]), batch 256 per GPU",
                   "model": "resnet50", "global_batch": world * B, "per_gpu_batch": B, "seq_len": 0,
                   "parallelism": f"dp{world} (batch-sharded, no collective for inference)",
                   "l2": "per-step working set >> 126 MB L2 (no flush needed)"},
        "e2e": {"value": e2e, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "source": "pinned host slots filled in place (input_buffers), H2D pipelined on the copy stream"},
        "e2e_sync_call": {"value": world * B / (sync_ms / 1e3), "unit": "images/s",
                          "api": "predict(numpy batch) per step: host copy into pinned + H2D + plan + D2H + sync, wall clock"},
        "gpus_active": gpus_active,
        "roofline": roof, "roofline_dfp": roof_dfp, "cpu_baseline": cpu, "clocks": clocks,
        "gpu_launches": launches_per_step * args.steps,
        "family_ms_per_step": {k: round(v / 1e3, 3) for k, v in sorted(fam_time.items(), key=lambda kv: -kv[1])[:8]},
        "train": train,
        "other_configs": others,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch this script as N ranks (one process per GPU)
    under torch.distributed.run on this node. Refuses when fewer than N GPUs are visible."""
    import socket
    if args.impl == "b200":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"bench: --gpus {args.gpus} requested but only {have} CUDA device(s) visible")
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


OTHER_CONFIGS = [
    # BASELINE.json configs beyond the headline (configs[2] inference, configs[3] training)
    ("configs[0] small CNN f32 inference B=32 32x32", "small_cnn", 32, "f32", 32),
    ("configs[1] ResNet-18 f32 (TF32 tensor cores) inference B=64 224x224", "resnet18", 64, "f32", 224),
    ("configs[4] DenseNet-121 bf16 inference B=128/GPU 224x224", "densenet121", 128, "bf16", 224),
    ("configs[4] MobileNet-V2 bf16 inference B=128/GPU 224x224", "mobilenet_v2", 128, "bf16", 224),
    ("configs[4] DenseNet-121 bf16 inference B=16/GPU (global 128 on 8 GPUs)", "densenet121", 16, "bf16", 224),
    ("configs[4] MobileNet-V2 bf16 inference B=16/GPU (global 128 on 8 GPUs)", "mobilenet_v2", 16, "bf16", 224),
]


def tf32_peak_tflops():
    """Dense TF32 tensor-core peak measured here (cuBLAS via torch.matmul, 8192^3, best of 5): the
    roofline denominator for the f32/TF32 configs (MEASURED_PEAKS.json has bf16 only)."""
    import torch
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device="cuda")
        b = torch.randn(n, n, device="cuda")
        for _ in range(2):
            a @ b
        best = 0.0
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            a @ b
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
        return best
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


def other_configs(args, peaks, peaks_kind, device):
    """Every other BASELINE config at full size on this GPU: device-timed images/s (inputs resident,
    CUDA events on the plan stream) and the conv / DFP rooflines of each plan."""
    from paper_2003_10688_b200 import frontend, models
    out = []
    tf32 = tf32_peak_tflops()
    for name, model, B, dt, hw in OTHER_CONFIGS:
        t0 = time.time()
        try:
            g = models.MODELS[model](hw=hw) if model == "small_cnn" else models.MODELS[model]()
            m = frontend.optimize(g, frontend.OptimizeOptions(batch=B, dtype=dt, device=device, fuse_epilogue=True))
            x = np.random.default_rng(7).uniform(-1, 1, (B, 3, hw, hw)).astype(np.float32)
            m.set_inputs({"x": x})
            for _ in range(max(args.warmup, 3)):
                m.run()
            m.sync()
            k = max(3, min(args.steps, 10))
            m.event(0)
            for _ in range(k):
                m.run()
            m.event(1)
            m.sync()
            ms = m.elapsed_ms(0, 1) / k
            pk = dict(peaks)
            if dt == "f32":
                pk["bf16_tflops_sustained"] = tf32  # TF32 tensor cores
            conv = {f for f in (st.family for st in m.steps) if f.startswith(("conv_", "linear"))}
            roof, _ = roofline_of(m, pk, peaks_kind if dt == "bf16" else "measured here (TF32 cuBLAS 8192^3)",
                                  conv, "tensor")
            dfp = {st.family for st in m.steps if st.family.startswith("dfp_")}
            roof_d, _ = roofline_of(m, pk, peaks_kind, dfp, "hbm") if dfp else (None, None)
            out.append({"workload": name, "value": B / (ms / 1e3), "unit": "images/s", "ms_per_step": ms,
                        "per_gpu_batch": B, "dtype": dt if dt == "bf16" else "f32 (TF32 tensor cores)",
                        "roofline_conv": roof, "roofline_dfp": roof_d, "units": len(m.units),
                        "compile_s": round(time.time() - t0, 1)})
            del m
        except Exception as e:  # reported, never silently dropped
            out.append({"workload": name, "error": f"{type(e).__name__}: {e}"})
    return {"tf32_peak_tflops_measured": tf32, "configs": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--train-batch", type=int, default=128)
    ap.add_argument("--train-steps", type=int, default=10)
    ap.add_argument("--no-train", dest="train", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", dest="configs", action="store_false",
                    help="skip the other BASELINE configs (small CNN, ResNet-18 TF32, DenseNet-121, MobileNet-V2)")
    args = ap.parse_args()
    if os.environ.get("SOL_BENCH_WATCHDOG"):  # diagnostics: dump every thread's stack if a run stalls
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["SOL_BENCH_WATCHDOG"]), repeat=False)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
