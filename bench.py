#!/usr/bin/env python
"""Benchmark of the integral-image scatterplot regularizer (BASELINE.json metric:
"regularization iters/sec (1M pts, 1024^2 grid); integral-image GB/s vs HBM peak").

N = 1 (default): BASELINE configs[1], the paper's Fig. 5 case: 1,000,000 points in
four Gaussian clusters (400k/300k/200k/100k, sigma 0.05, centres at 0.3/0.7),
float32-representable, on a 1024^2 grid, kernel_size 8, 10 iterations.  One "step" is
one full 10-iteration regularization of that input, device resident (inputs already in
HBM).  L2 is flushed (256 MiB write) between timed steps.  The line also carries the
integral-image pass (configs[4] at 4096^2 and 16384^2) and the SPLOM batch on this one
GPU (configs[3], the N = 1 point of the scaling curve).

N > 1: BASELINE configs[3], the SPLOM batch (256 plots x 500k points, 1024^2, 10
iterations) sharded over N GPUs (strong scaling): each rank runs its block of plots as
one batched run, and the step ends with one NCCL all-gather of every plot's final
positions.  `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload ...]

`--impl reference` times the reference algorithm's CPU implementation (the C port in
oracle/, all host threads) on the same workload and config; rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_POINTS = 1_000_000
K_GRID = 10
KERNEL_SIZE = 8
ITERS = 10
METRIC = "regularization iters/sec (1M pts, 1024² grid); integral-image GB/s vs HBM peak"


def four_cluster(n: int = N_POINTS, seed: int = 4) -> np.ndarray:
    """Four Gaussian clusters (0.4/0.3/0.2/0.1 of n, sigma 0.05, centres 0.3/0.7),
    resampled until inside [0,1]^2, rounded to float32-representable values."""
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = ((0.3, 0.3), (0.7, 0.3), (0.3, 0.7), (0.7, 0.7))
    counts = [n * 4 // 10, n * 3 // 10, n * 2 // 10]
    counts.append(n - sum(counts))
    parts = []
    for c, m in zip(centres, counts):
        p = rng.normal(c, 0.05, size=(m, 2))
        for _ in range(64):
            bad = np.any((p < 0) | (p > 1), axis=1)
            if not bad.any():
                break
            p[bad] = rng.normal(c, 0.05, size=(int(bad.sum()), 2))
        parts.append(np.clip(p, 0, 1))
    return np.concatenate(parts).astype(np.float32).astype(np.float64)


def c3_points(n: int, seed: int = 42) -> np.ndarray:
    """BASELINE configs[2] input: gaussian mixture of 4-8 clusters, sigma 0.02-0.06
    (the reference acceptance-test pattern), fp32-representable."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence((seed, n))))
    m = int(rng.integers(4, 9))
    w = rng.uniform(0.5, 2.0, size=m)
    counts = np.floor(w / w.sum() * n).astype(np.int64)
    counts[: n - int(counts.sum())] += 1
    centres = rng.uniform(0.12, 0.88, size=(m, 2))
    sig = rng.uniform(0.02, 0.06, size=m)
    parts = []
    for c in range(m):
        p = rng.normal(centres[c], sig[c], size=(int(counts[c]), 2))
        for _ in range(64):
            bad = np.any((p < 0) | (p > 1), axis=1)
            if not bad.any():
                break
            p[bad] = rng.normal(centres[c], sig[c], size=(int(bad.sum()), 2))
        parts.append(np.clip(p, 0, 1))
    return np.concatenate(parts).astype(np.float32).astype(np.float64)


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons through NVML during the timed region."""

    def __init__(self, index: int, period: float = 0.001):
        super().__init__(daemon=True)
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.stop_flag = threading.Event()
        self.max_mhz = None
        self.ok = False

    def run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
                "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
            }
            self.ok = True
            while not self.stop_flag.is_set():
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for nm, bit in names.items():
                    if r & bit and nm != "gpu_idle":
                        self.reasons.add(nm)
                time.sleep(self.period)
        except Exception as e:  # NVML missing: report it rather than inventing clocks
            self.reasons.add(f"nvml_unavailable:{type(e).__name__}")

    def summary(self):
        self.stop_flag.set()
        self.join(timeout=2)
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# Algorithmic bytes per launch of each kernel,
# n points, m = s^2 pixels.
def algorithmic_bytes(name: str, n: int, m: int) -> int:
    """Minimal DRAM bytes per launch of each kernel of the iteration (n points, m pixels);
    DESIGN.md section 4.  Grid-sized aggregates (1/TH of the grid) are left out."""
    table = {
        "splat": 8 * n + 4 * m,            # read fp32 (x,y); counts written once
        "smooth_h": 4 * m + 4 * m + 4 * m,  # read counts, write the horizontal pass, clear the next counts
        "smooth_v_reduce": 4 * m + 4 * m,  # read the horizontal pass, write d
        "write_field": 4 * m + 8 * m,      # read d, write the (s,s,2) field once
        "sample": 16 * n + 8 * m + 4 * m,  # read + write fp32 points, field gathered once, next counts written once
        "memset_counts": 8 * m,
    }
    return table.get(name, 0)


# ncu kernel names -> the names inim_profile_run reports
NCU_NAMES = {"sample_f32_kernel": "sample", "move_bulk_kernel": "sample", "write_kernel": "write_field", "smooth_h_kernel": "smooth_h",
             "smooth_v_kernel": "smooth_v_reduce", "chains_kernel": "chains", "splat_f32_kernel": "splat",
             "lines_kernel": "lines", "chains_reg_kernel": "chains"}


def ncu_traffic(workload: str):
    """Per-launch DRAM bytes (read + write) of each kernel from the committed ncu launch
    list of this workload (profiles/traffic_<workload>.json, tools/traffic_json.py), or {}."""
    f = Path(__file__).resolve().parent / "profiles" / f"traffic_{workload}.json"
    if not f.exists():
        return {}
    try:
        return json.loads(f.read_text()).get("per_launch_bytes", {})
    except ValueError:
        return {}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world: int, backend: str):
    import torch.distributed as dist

    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return dist


SPLOM_POINTS = 500_000
SPLOM_METRIC = "regularization iters/sec (SPLOM batch, 500k pts per plot, 1024² grid)"
SPLOM_BYTES_PER_PLOT_ITER = 37.2e6  # 24 n + 24 m bytes at n = 500k, m = 1024^2


def c2_config(world: int) -> dict:
    """The config dict of the C2 line (identical in both arms)."""
    return {"workload": "1M pts, 1024^2 grid, kernel_size 8, 10 iterations per step (BASELINE configs[1])",
            "points": N_POINTS, "grid": 1 << K_GRID, "iterations_per_step": ITERS, "kernel_size": KERNEL_SIZE,
            "input": "four_cluster(1M, seed=4)", "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"replicas x{world}" if world > 1 else "single plot"}


def c3_config(world: int) -> dict:
    return {"workload": "16M pts, 4096^2 grid, kernel_size 8, 10 iterations per step (BASELINE configs[2])",
            "points": 16_000_000, "grid": 4096, "iterations_per_step": ITERS, "kernel_size": KERNEL_SIZE,
            "input": "c3_points(16M, seed=42)", "l2": "flushed between timed steps (256 MiB write)",
            "parallelism": f"replicas x{world}" if world > 1 else "single plot"}


def splom_config(world: int, plots: int) -> dict:
    return {"workload": f"SPLOM {plots} plots x 500k pts, 1024^2, kernel_size 8, 10 iterations (BASELINE configs[3])",
            "plots": plots, "points_per_plot": SPLOM_POINTS, "grid": 1 << K_GRID, "iterations_per_step": ITERS,
            "kernel_size": KERNEL_SIZE, "input": "splom_plot(idx, 500k), PCG64 seeds (2408, idx)",
            "parallelism": f"plots sharded over {world} GPU(s) (contiguous blocks), one batched run per rank, "
                           "NCCL all-gather of the final positions inside the step",
            "l2": "flushed between timed steps (256 MiB write)"}


# ------------------------------------------------------------------------ our arm
def bench_ours(args):
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist = init_dist(world, "nccl")
    import paper_2408_06513_b200 as P
    from paper_2408_06513_b200 import _device as D
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda", local)
    if args.workload == "c3":
        host, k = c3_points(16_000_000, seed=42 + rank), 12
    else:
        host, k = four_cluster(N_POINTS, seed=4 + rank), K_GRID
    n = len(host)
    m = 1 << (2 * k)
    pts_in = torch.from_numpy(host.astype(np.float32)).to(dev)
    pts = torch.empty_like(pts_in)
    ws = torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    gathered = torch.empty((world, n, 2), dtype=torch.float32, device=dev) if world > 1 else None
    stream = D.stream()

    def step():
        pts.copy_(pts_in)
        _lib.check(lib.inim_run(D.ptr(pts), n, k, KERNEL_SIZE, 0.0, ITERS, 0.0, None, None, None, None, None,
                                D.ptr(ws), stream), "inim_run")
        if gathered is not None:
            dist.all_gather_into_tensor(gathered, pts)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for q in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (256 MiB > 126 MB L2), outside the step events
        starts[q].record()
        step()
        ends[q].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.summary()
    t_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if world > 1:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    value = world * ITERS * args.steps / (t_ms / 1e3)

    # -- per-kernel attribution: eager launches with an event after each launch
    cap = 64 * ITERS
    ms = (ctypes.c_float * cap)()
    names = ctypes.create_string_buffer(cap * 24)
    per_kernel: dict = {}
    prof_steps = 3
    for _ in range(prof_steps):
        flush.zero_()
        pts.copy_(pts_in)
        cnt = lib.inim_profile_run(D.ptr(pts), n, k, KERNEL_SIZE, 0.0, ITERS, D.ptr(ws), stream, ms, cap, names,
                                   len(names))
        if cnt < 0:
            _lib.check(cnt, "profile_run")
        for nm, v in zip(names.value.decode().split("\n")[:cnt], ms[:cnt]):
            e = per_kernel.setdefault(nm, [0.0, 0])
            e[0] += v
            e[1] += 1
    prof_total = sum(v[0] for v in per_kernel.values()) / prof_steps
    kernels = {nm: {"avg_us": 1e3 * v[0] / v[1], "launches_per_step": v[1] // prof_steps,
                    "share": (v[0] / prof_steps) / prof_total} for nm, v in per_kernel.items()}
    dom = max((nm for nm in kernels if nm != "memset_counts"), key=lambda nm: kernels[nm]["share"])
    peaks = measured_peaks()
    dom_bytes = algorithmic_bytes(dom, n, m)
    achieved = dom_bytes / (kernels[dom]["avg_us"] * 1e-6) / 1e9 if dom_bytes else None

    # -- integral-image pass alone (BASELINE configs[4] at 4096^2 and 16384^2), L2 flushed
    integral = bench_integral(lib, D, dev, flush, sizes=(12, 14), reps=10)

    # -- end to end through the public API with host buffers (pinned), rank-local
    e2e = bench_e2e(P, host, k, reps=max(3, min(args.steps, 10)))

    # -- the SPLOM batch (configs[3]) on this GPU: the N = 1 point of the scaling curve
    splom = None
    if world == 1 and not args.no_splom and args.workload in (None, "c2"):
        splom = bench_splom(args, emit=False)
        for key in ("config", "data", "clocks", "vs_baseline", "higher_is_better", "dtype"):
            splom.pop(key, None)

    if rank != 0:
        return
    cpu = cpu_baseline(host, k, iterations=4 if k == K_GRID else 2) \
        if world == 1 and not args.no_cpu_baseline else None
    c3 = args.workload == "c3"
    line = {
        "metric": METRIC if not c3 else "regularization iters/sec (16M pts, 4096² grid)",
        "value": value,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": ("synthetic gaussian mixture (4-8 clusters, sigma 0.02-0.06), fp32-representable" if c3 else
                 "synthetic four-cluster (400k/300k/200k/100k, sigma 0.05), fp32-representable"),
        "config": c3_config(world) if c3 else c2_config(world),
        "e2e": e2e,
        # (the point sort's mark spans three kernels: block sums, block scans, placement)
        "gpu_launches": int(args.steps * sum(v["launches_per_step"] * (3 if nm == "sort_points" else 1)
                                             for nm, v in kernels.items() if nm != "memset_counts")),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": (achieved / peaks["hbm_gbs"]) if achieved else None,
                     "traffic": ncu_traffic("c3" if c3 else "c2").get(dom),
                     "traffic_source": f"profiles/traffic_{'c3' if c3 else 'c2'}.json (ncu dram__bytes_read+write "
                                       "per launch, cold cache)",
                     "algorithmic_bytes_per_launch": dom_bytes, "avg_launch_us": kernels[dom]["avg_us"],
                     "peak_source": peaks["source"],
                     "method": "per-launch CUDA events on the launch stream (eager replay of the timed step)"},
        "kernels": kernels,
        "integral_image": integral,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "splom_1gpu": splom,
    }
    print(json.dumps(line), flush=True)


def bench_integral(lib, D, dev, flush, sizes=(12,), reps=10):
    """inim_integral_set GB/s on random fp32 textures, 36 B/px algorithmic."""
    import torch
    from paper_2408_06513_b200 import _lib

    peaks = measured_peaks()
    out = []
    for k in sizes:
        s = 1 << k
        g = torch.Generator(device=dev)
        g.manual_seed(1234)
        d = torch.rand((s, s), generator=g, device=dev, dtype=torch.float32) * 10.0
        tables = torch.empty((8, s, s), dtype=torch.float32, device=dev)
        total = torch.empty(1, dtype=torch.float64, device=dev)
        ws = torch.empty(int(lib.inim_workspace_bytes(k, 0, 1)), dtype=torch.uint8, device=dev)
        st = D.stream()

        def once():
            _lib.check(lib.inim_integral_set(D.ptr(d), k, D.ptr(tables), D.ptr(total), D.ptr(ws), st), "integral")

        for _ in range(3):
            once()
        times = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            once()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b))
        t = statistics.median(times) / 1e3
        gbs = 36 * s * s / t / 1e9
        out.append({"size": s, "ms": t * 1e3, "GB_s": gbs, "frac": gbs / peaks["hbm_gbs"],
                    "bytes_per_px": 36, "l2": "flushed"})
        del d, tables, ws
    return out


def bench_e2e(P, host: np.ndarray, k: int, reps: int):
    """Same metric through the public drop-in API with host (pinned) buffers: H2D of the
    float64 positions, 10 device iterations, D2H of the final frame, every call."""
    import torch

    n = len(host)
    pinned = torch.empty((n, 2), dtype=torch.float64).pin_memory()
    pinned.numpy()[:] = host
    pos = pinned.numpy()
    params = P.RegularizationParams(k=k, kernel_size=KERNEL_SIZE, iterations=ITERS, frame_cap=2)

    def call():
        r = P.run(P.ScatterDataset(positions=pos), params, store_fields=False)
        return r.frame(ITERS)

    for _ in range(3):
        call()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(reps, 10)):
        t0 = time.perf_counter()
        out = call()  # returns host float64: the call has synchronised
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    assert out.shape == (n, 2)
    return {"value": ITERS / dt, "unit": "iters/s", "h2d_bytes_per_step": int(n * 2 * 8),
            "d2h_bytes_per_step": int(n * 2 * 8), "ms_per_call": dt * 1e3,
            "ms_per_call_min_max": [min(times) * 1e3, max(times) * 1e3], "calls": len(times),
            "statistic": "median wall time per call",
            "api": f"paper_2408_06513_b200.run(ScatterDataset, RegularizationParams(k={k}, kernel_size=8, "
                   "iterations=10, frame_cap=2), store_fields=False).frame(10)"}


# ------------------------------------------------------------------ CPU baseline
def cpu_baseline(host: np.ndarray, k: int = K_GRID, iterations: int = 4):
    """The oracle (C restatement of the reference algorithm, float64) with every host
    thread, on a bounded sample: `iterations` iterations of the same input and grid."""
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    O.set_threads(cores)
    defect = O.flat_response(k)
    pos = host
    t0 = time.perf_counter()
    for _ in range(iterations):
        pos = O.iterate_once(pos, k, KERNEL_SIZE, None, defect)
    dt = time.perf_counter() - t0
    return {"value": iterations / dt, "unit": "iters/s", "cores": cores, "kind": "port",
            "sample": f"{iterations} iterations of the {len(host)}-point / {1 << k}^2 / ks=8 workload (float64 C "
                      f"port of the reference algorithm, OpenMP {cores} threads)"}


def bench_reference(args, workload: str):
    """The reference arm: the reference algorithm's CPU implementation (the C port in
    oracle/, every host thread) on our arm's workload, config, metric and unit; each
    step is a bounded sample of that workload.  Rank 0 only."""
    rank, world, _local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    O.set_threads(cores)
    defect = O.flat_response(K_GRID)
    if workload == "splom":
        from paper_2408_06513_b200.splom import splom_plot

        plots = [splom_plot(i, SPLOM_POINTS) for i in range(2)]
        metric, unit, config = SPLOM_METRIC, "plot-iters/s", splom_config(world, args.plots)
        sample = (f"each step = 1 iteration of one 500k-point / 1024^2 / ks=8 SPLOM plot (plots 0 and 1 "
                  f"alternating); float64 C port of the reference algorithm, OpenMP {cores} threads")

        def step(q, pos):
            return O.iterate_once(pos[q % 2], K_GRID, KERNEL_SIZE, None, defect)

        state = plots
    else:
        host = four_cluster(N_POINTS, seed=4)
        metric, unit, config = METRIC, "iters/s", c2_config(world)
        sample = (f"each step = 1 iteration of the 1M-point / 1024^2 / ks=8 workload (the timed unit of our arm is "
                  f"10 iterations); float64 C port of the reference algorithm, OpenMP {cores} threads")

        def step(q, pos):
            return O.iterate_once(pos, K_GRID, KERNEL_SIZE, None, defect)

        state = host
    for q in range(args.warmup):
        out = step(q, state)
        if workload != "splom":
            state = out
    state = plots if workload == "splom" else host
    t0 = time.perf_counter()
    for q in range(args.steps):
        out = step(q, state)
        if workload != "splom":
            state = out
    dt = time.perf_counter() - t0
    value = args.steps / dt
    line = {
        "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if workload == "splom" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic, fp32-representable (same generators as our arm)", "config": config,
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": unit, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class _StubSplom:
    """CPU stand-in for DeviceSplom (--cpu-stub): the same shard / chunked run /
    pipelined gather plumbing with the per-plot compute replaced by a deterministic
    transform, so the multi-rank path of this file runs on gloo without a GPU
    (tests/test_distributed.py)."""

    def __init__(self, ids, points, batch):
        import torch

        self.ids = list(ids)
        self.work = torch.zeros((len(self.ids), points, 2), dtype=torch.float32)
        self.chunks = [(b0, min(b0 + batch, len(self.ids))) for b0 in range(0, len(self.ids), batch)]

    def run(self, on_chunk=None):
        for b0, b1 in self.chunks:
            for q in range(b0, b1):
                self.work[q].fill_(float(self.ids[q]))
            if on_chunk is not None:
                on_chunk(b0, b1)
        return self.work


def splom_job(args, world: int, rank: int, device_stub: bool):
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, pipeline_parts, shard, splom_plot

    ids = shard(args.plots, world, rank)
    points = args.splom_points
    # with a pipelined gather the block runs as sub-batches of the pipeline's width
    batch = pipeline_parts(args.plots, world, args.gather_parts)[0][1] if world > 1 else args.plots
    if device_stub:
        return _StubSplom(ids, points, max(1, batch)), ids
    cfg = SplomConfig(nplots=args.plots, points=points, k=K_GRID, kernel_size=KERNEL_SIZE, iterations=ITERS,
                      max_batch=max(1, batch))
    job = DeviceSplom(cfg, ids)
    job.load(lambda i: splom_plot(i, points))
    return job, ids


def bench_splom(args, emit: bool = True):
    """BASELINE configs[3]: SPLOM of --plots plots x 500k points, 1024^2, 10 iterations,
    plots sharded over ranks (one batched run per rank), one NCCL all-gather of the
    final positions inside the step.  value = plot-iterations per second (whole job),
    time = max over ranks of the device-timed steps.  With emit=False (the N = 1 C2
    line) returns the measurement instead of printing it."""
    import torch

    rank, world, local = dist_env()
    stub = args.cpu_stub
    if not stub:
        torch.cuda.set_device(local)
    dist = init_dist(world, "gloo" if stub else "nccl")
    from paper_2408_06513_b200.splom import GatherPipeline

    job, ids = splom_job(args, world, rank, stub)
    flush = None if stub else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    gathered = {}

    def step():
        if world == 1:
            gathered["all"] = job.run()
            return
        # each sub-batch's all-gather starts as soon as its batched run is enqueued and
        # overlaps the next sub-batch's compute
        pipe = GatherPipeline(args.plots, world, rank, args.gather_parts, job.work)
        job.run(on_chunk=lambda b0, b1: pipe.ready(job.work, b1))
        gathered["all"] = pipe.finish(job.work)

    def sync():
        if not stub:
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    sync()
    sampler = None
    if not stub:
        sampler = ClockSampler(local)
        sampler.start()
    if world > 1:
        dist.barrier()
    sync()
    t_ms = 0.0
    for _ in range(args.steps):
        if stub:
            t0 = time.perf_counter()
            step()
            t_ms += (time.perf_counter() - t0) * 1e3
            continue
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        b.synchronize()
        t_ms += a.elapsed_time(b)
    sync()
    if world > 1:
        dist.barrier()
    clocks = sampler.summary() if sampler else None
    if world > 1:
        t = torch.tensor([t_ms], dtype=torch.float64, device="cpu" if stub else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    allres = gathered["all"]
    gather_ok = bool(allres.shape[0] == args.plots)
    if stub:  # every plot's block came back in order
        gather_ok = gather_ok and all(float(allres[i, 0, 0]) == float(i) for i in range(args.plots))
    e2e = None if stub else splom_e2e(args, job, world, dist)
    total_iters = args.plots * ITERS * args.steps
    value = total_iters / (t_ms / 1e3)
    peaks = measured_peaks()
    achieved = SPLOM_BYTES_PER_PLOT_ITER * value / 1e9
    launches = None if stub else int(args.steps * job_launches(job))
    out = {
        "metric": SPLOM_METRIC, "value": value, "unit": "plot-iters/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": ("CPU stub (per-plot compute replaced; plumbing test only)" if stub else
                 "synthetic gaussian mixtures (PCG64 seeds (2408, plot)), fp32-representable"),
        "config": splom_config(world, args.plots),
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "kernel": "whole iteration (all stages, batched)", "achieved": achieved,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                     "traffic": None, "peak_source": peaks["source"],
                     "algorithmic_bytes_per_plot_iteration": SPLOM_BYTES_PER_PLOT_ITER,
                     "method": "24 n + 24 m bytes per plot-iteration (SURVEY 8(d)) x plot-iterations / s"},
        "collective": {"backend": dist.get_backend() if world > 1 else None, "world": world,
                       "op": (f"all_gather_into_tensor of final positions in {args.gather_parts} sub-batches, each "
                              "overlapping the next sub-batch's compute") if world > 1 else None,
                       "bytes_per_step": int(args.plots * args.splom_points * 8) if world > 1 else 0,
                       "gather_ok": gather_ok},
        "plots_per_rank": len(ids),
        "clocks": clocks,
    }
    if not emit:
        return out
    if rank == 0:
        print(json.dumps(out), flush=True)
    return out


def job_launches(job) -> int:
    """Kernels per SPLOM step: per batched run, the splat, the point sort (block sums,
    block scans with their own prefix, placement), six kernels per iteration and the
    final unpermute (+ the counts memset node, not a kernel)."""
    return len(job.chunks) * (1 + 3 + 6 * ITERS + 1)


def splom_e2e(args, job, world, dist):
    """The same step through the public API with host buffers: every rank runs its
    block of plots from page-locked host memory (float32, as the batch API takes them)
    with DeviceSplom.run_host, whose chunked copies in and out overlap the batched runs,
    and holds its block of final positions on the host; time = max over ranks."""
    import torch

    host_in = torch.empty(tuple(job.inputs.shape), dtype=torch.float32).pin_memory()
    host_in.copy_(job.inputs.cpu())
    host_out = torch.empty_like(host_in).pin_memory()

    def call():
        job.run_host(host_in, host_out)
        torch.cuda.current_stream().synchronize()

    for _ in range(2):
        call()
    times = []
    for _ in range(max(3, min(args.steps, 5))):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    nbytes = int(host_in.numel() * 4)
    return {"value": args.plots * ITERS / dt, "unit": "plot-iters/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "ms_per_call": dt * 1e3, "statistic": "median wall time, max over ranks",
            "api": "DeviceSplom.run_host (chunked H2D / inim_run_batched / D2H overlapped on three streams), "
                   "pinned float32 host buffers, each rank its own block"}


def bench_sweep(args):
    """BASELINE configs[4]: integral-image-only sweep 512^2 .. 16384^2, fp32, L2 flushed."""
    import torch

    from paper_2408_06513_b200 import _device as D
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    sampler = ClockSampler(0)
    sampler.start()
    rows = bench_integral(lib, D, dev, flush, sizes=tuple(range(9, 15)), reps=max(5, args.steps))
    clocks = sampler.summary()
    best = max(rows, key=lambda r: r["frac"])
    line = {"metric": "integral-image GB/s vs HBM peak (36 B/px: read d, write 8 fp32 tables)",
            "value": best["GB_s"], "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": 3,
            "ms_per_step": best["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic uniform random textures",
            "config": {"workload": "integral-image-only sweep 512^2..16384^2 (BASELINE configs[4])",
                       "best_size": best["size"]},
            "sweep": rows, "clocks": clocks}
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch(args) -> int:
    """`--gpus N` outside torchrun: run this file under torch.distributed.run with N
    ranks (one per GPU) and pass its exit code through."""
    import subprocess

    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # NCCL prints nranks per communicator: the rank count is on record
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["c2", "c3", "splom", "sweep"],
                    help="default: c2 (1M pts/1024^2, the headline) on one GPU, splom (configs[3]) on N > 1; "
                         "c3: 16M pts/4096^2; sweep: integral-only 512^2..16384^2")
    ap.add_argument("--plots", type=int, default=256)
    ap.add_argument("--splom-points", type=int, default=SPLOM_POINTS)
    ap.add_argument("--gather-parts", type=int, default=2, help="N > 1: sub-batches of the pipelined gather")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-splom", action="store_true", help="N = 1: leave the SPLOM batch out of the C2 line")
    ap.add_argument("--cpu-stub", action="store_true", help="multi-rank plumbing on gloo, no GPU (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank, world, _ = dist_env()
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    workload = args.workload or ("c2" if world == 1 else "splom")
    if args.impl == "reference":
        bench_reference(args, workload)
    elif args.cpu_stub:
        bench_splom(args)
    elif workload == "splom":
        bench_splom(args)
    elif workload == "sweep":
        bench_sweep(args)
    else:
        bench_ours(args)
    if world > 1:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
