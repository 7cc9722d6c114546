"""Iterative density equalization on the GPU (drop-in for uncrowd regularize.py:25-109).

``run`` keeps every iteration on the device: the positions are narrowed to float32
once, then chunks of iterations are replayed as one CUDA graph each (inim_run:
counts <- 0, splat, smoothing + tile reduce, carry scan, fused integral/field,
bilinear move + clip).  The host only records the frames the reference's frame_cap
policy keeps and reads the displacement-stop state between chunks.
"""

from __future__ import annotations

import time
from typing import Optional

import numpy as np
import torch

from . import _device as D
from . import _lib
from .density import build_density, resolve_background
from .errors import OutOfRangeLevel
from .mapping import _defect_device, flat_response, sample_points
from .metrics import RunMetrics, record_for_frame
from .model import DeformationField, RegularizationParams, RegularizationRun, ScatterDataset

CHUNK = 16  # iterations per captured graph


def iterate_once(positions: np.ndarray, params: RegularizationParams, defect: Optional[np.ndarray] = None):
    """One equalization step: (new positions, field, density) (regularize.py:25-37).

    Float64 positions are binned in float64 (bit-exact counts for identical inputs)
    and moved with float64 bilinear weights; density and field are float32 on the
    device.  Sample order is preserved.
    """
    lib = D.require_cuda()
    density = build_density(positions, params)
    if defect is None:
        flat_response.touch(params.k)  # the closed form is evaluated in the field kernel
    k = params.k
    s = 1 << k
    dev_def = _defect_device(k, defect, torch.float32)
    targets = torch.empty((s, s, 2), dtype=torch.float32, device=D.device())
    exc = torch.zeros(1, dtype=torch.float32, device=D.device())
    total = torch.empty(1, dtype=torch.float64, device=D.device())
    ws = D.workspace(k)
    _lib.check(lib.inim_field_from_density(D.ptr(density.device_values()), k, D.ptr(dev_def), D.ptr(targets),
                                           D.ptr(exc), D.ptr(total), D.ptr(ws), D.stream()), "iterate_once")
    field = DeformationField(k=k, max_excursion=float(exc.item()), device_targets=targets)
    new_positions = sample_points(field, positions, clip=True)
    return new_positions, field, density


def _device_iterate(pos: torch.Tensor, params: RegularizationParams, n: Optional[int] = None, with_field=True):
    """One float32 device iteration (the run loop's own step): (new positions, field).
    Used by stop="time" and to recompute frames thinned away by frame_cap.  Same kernels
    as inim_run: bit-identical.  `n` (default: all rows of `pos`) may be 0 with a
    one-row placeholder `pos`."""
    lib = D.require_cuda()
    if n is None:
        n = pos.shape[0]
    k = params.k
    bufs = _run_buffers(n, k, 1, False)
    out = torch.empty_like(pos)
    bg = resolve_background(params, n)
    _lib.check(lib.inim_iterate(D.ptr(pos), D.ptr(out), n, k, params.kernel_size, bg, None, D.ptr(bufs["counts"]),
                                D.ptr(bufs["d"]), D.ptr(bufs["targets"]), D.ptr(bufs["exc"]), D.ptr(bufs["disp"]),
                                0.0, None, D.ptr(bufs["ws"]), D.stream()), "iterate")
    if not with_field:
        return out, None
    field = DeformationField(k=k, max_excursion=float(bufs["exc"].item()), device_targets=bufs["targets"].clone())
    return out, field


_bufcache: dict = {}


def _run_buffers(n: int, k: int, chunk: int, store_fields: bool):
    """Persistent device buffers per (n, k, chunk, store_fields): graph replays need
    stable pointers."""
    D.check_grid(k)
    key = (torch.cuda.current_device(), n, k, chunk, store_fields)
    b = _bufcache.get(key)
    if b is None:
        lib = D.require_cuda()
        s = 1 << k
        dev = D.device()
        b = {
            "ws": torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device=dev),
            "pts": torch.empty((max(n, 1), 2), dtype=torch.float32, device=dev),
            "frames": torch.empty((chunk + 1, max(n, 1), 2), dtype=torch.float32, device=dev),
            "fields": torch.empty((chunk, s, s, 2), dtype=torch.float32, device=dev) if store_fields else None,
            "disp": torch.zeros(chunk, dtype=torch.float32, device=dev),
            "excs": torch.zeros(chunk, dtype=torch.float32, device=dev),
            "state": torch.zeros(4, dtype=torch.int32, device=dev),
            "counts": torch.empty((s, s), dtype=torch.int32, device=dev),
            "d": torch.empty((s, s), dtype=torch.float32, device=dev),
            "targets": torch.empty((s, s, 2), dtype=torch.float32, device=dev),
            "exc": torch.zeros(1, dtype=torch.float32, device=dev),
        }
        if len(_bufcache) > 8:
            torch.cuda.synchronize()
            lib.inim_clear_graph_cache()
            _bufcache.clear()
        _bufcache[key] = b
    return b


def _survivors(iterations: int, frame_cap: int) -> set:
    """Frames the reference's thinning policy (model.py:155-162) keeps after a fixed
    number of iterations."""
    kept, stride = {0}, 1
    for t in range(1, iterations + 1):
        kept.add(t)
        if len(kept) > frame_cap:
            stride *= 2
            kept = {i for i in kept if i in (0, t) or i % stride == 0}
    return kept


def run(dataset: ScatterDataset, params: RegularizationParams, collect_metrics: str = "none",
        store_fields: bool = True, n_neighbors: int = 10) -> RegularizationRun:
    """Repeat iterations until the stopping criterion fires (regularize.py:40-80)."""
    params.validate()
    lib = D.require_cuda()
    result = RegularizationRun(dataset, params, store_fields=store_fields)
    flat_response.touch(params.k)  # built once per k, as the reference (regularize.py:51); the device
    # iteration evaluates the closed form in registers, so the arrays stay unmaterialised
    n = dataset.n
    k = params.k
    bg = resolve_background(params, n)
    metrics = collect_metrics != "none"
    full = collect_metrics == "full"
    if metrics:  # frame 0 (regularize.py:53-57)
        result.metrics.append(record_for_frame(0, dataset.positions, dataset.positions, k, wall_ms=0.0, full=full,
                                               n_neighbors=n_neighbors))
    if params.iterations == 0:
        return result
    if params.stop == "time":
        return _run_timed(result, dataset, params, bg, collect_metrics, n_neighbors)

    chunk = min(CHUNK, params.iterations)
    b = _run_buffers(n, k, chunk, store_fields)
    rm = RunMetrics(dataset.positions, k, chunk, full, n_neighbors) if metrics and n else None
    pts = b["pts"][:n] if n else b["pts"]
    if n:
        D.to_device(dataset.positions, out=pts)
    state = b["state"]
    state.zero_()
    eps = float(params.epsilon) if params.stop == "displacement" else 0.0
    if eps > 0.0:
        # the device compares float32 displacements: a positive epsilon below the smallest
        # float32 denormal must not round to 0 (which would disable the criterion)
        eps = max(float(np.float32(eps)), float(np.finfo(np.float32).smallest_subnormal))
    keep = _survivors(params.iterations, params.frame_cap) if params.stop == "fixed" else None
    done = 0
    early = None
    stream = D.stream()
    start_ev = torch.cuda.Event(enable_timing=True)
    end_ev = torch.cuda.Event(enable_timing=True)
    while done < params.iterations:
        c = min(chunk, params.iterations - done)
        # per-iteration frames only when the thinning policy keeps one inside the chunk;
        # the chunk's last frame is the point buffer itself
        frames_needed = keep is None or any((done + t) in keep for t in range(1, c))
        frames = b["frames"] if frames_needed else None
        start_ev.record()
        if rm is None:
            _lib.check(lib.inim_run(D.ptr(pts), n, k, params.kernel_size, bg, c, eps, D.ptr(frames),
                                    D.ptr(b["fields"]), D.ptr(b["disp"]), D.ptr(b["excs"]), D.ptr(state),
                                    D.ptr(b["ws"]), stream), "run")
        else:
            _lib.check(lib.inim_run_metrics(D.ptr(pts), n, k, params.kernel_size, bg, c, eps, D.ptr(frames),
                                            D.ptr(b["fields"]), D.ptr(b["disp"]), D.ptr(b["excs"]), D.ptr(state),
                                            D.ptr(b["ws"]), stream, *rm.args()), "run")
        end_ev.record()
        if eps == 0.0 and n and done + c == params.iterations:
            # the run's last frame is the point buffer: start its host copy before the
            # host waits, so it overlaps the bookkeeping below (frame() waits for it)
            early = D.to_host64_async(pts)
        end_ev.synchronize()
        per_iter = start_ev.elapsed_time(end_ev) / 1e3 / c
        if eps > 0:
            st = state.cpu().numpy()
            executed = int(st[1]) - done
            stopped = bool(st[0])
            if executed <= 0 and not stopped:
                raise RuntimeError("run: the device executed no iteration of a displacement-stop chunk")
        else:
            executed, stopped = c, False
        excs = b["excs"][:executed].cpu().numpy() if executed and store_fields else []
        for t in range(executed):
            it = done + t + 1
            result.wall_times.append(per_iter)
            if store_fields:
                result.fields.append(DeformationField(k=k, max_excursion=float(excs[t]),
                                                      device_targets=b["fields"][t].clone()))
            if keep is None or it in keep:
                src_frame = b["frames"][t + 1, :n] if frames is not None else pts
                result._record(it, src_frame.clone())
            else:
                result.iterations = it
        if metrics:
            if rm is not None:
                result.metrics.extend(rm.records(done + 1, executed, per_iter * 1e3))
            else:  # no samples: the reference's records of an empty layout
                result.metrics.extend(record_for_frame(done + t + 1, dataset.positions, dataset.positions, k,
                                                       wall_ms=per_iter * 1e3, full=full, n_neighbors=n_neighbors)
                                      for t in range(executed))
        done += executed
        if stopped:
            break
    if early is not None and result.iterations in result._dev_frames:
        result._pending[result.iterations] = early
    else:
        result._prefetch(result.iterations)
    return result


def _run_timed(result: RegularizationRun, dataset: ScatterDataset, params: RegularizationParams, bg: float,
               collect_metrics: str = "none", n_neighbors: int = 10):
    """stop='time': the budget is host wall time, checked between iterations
    (regularize.py:62-63), so iterations are launched one at a time."""
    n = dataset.n
    pos = D.to_device(dataset.positions).reshape(n, 2) if n else torch.zeros((1, 2), device=D.device())
    started = time.perf_counter()
    for t in range(1, params.iterations + 1):
        if time.perf_counter() - started > params.time_budget:
            break
        tick = time.perf_counter()
        new, field = _device_iterate(pos, params, n)
        torch.cuda.synchronize()
        wall = time.perf_counter() - tick
        result.wall_times.append(wall)
        if result.store_fields:
            result.fields.append(field)
        result._record(t, new if n else new[:0])
        if collect_metrics != "none":
            result.metrics.append(record_for_frame(t, dataset.positions, new if n else dataset.positions, params.k,
                                                   wall_ms=wall * 1e3, full=collect_metrics == "full",
                                                   n_neighbors=n_neighbors))
        pos = new
    return result


def transition_positions(run_result: RegularizationRun, level: float) -> np.ndarray:
    """Per-sample linear blend between the two frames bracketing `level`
    (regularize.py:83-93)."""
    top = run_result.iterations
    if not 0.0 <= level <= top:
        raise OutOfRangeLevel(f"level {level} outside [0, {top}]")
    low, high = int(np.floor(level)), int(np.ceil(level))
    if low == high:
        return run_result.frame(low)
    frac = level - low
    return (1.0 - frac) * run_result.frame(low) + frac * run_result.frame(high)


def map_through(fields, points: np.ndarray, upto: Optional[int] = None) -> np.ndarray:
    """Push points through the composed per-iteration fields (regularize.py:96-109).

    Fields produced by ``run`` are float32 device fields; points then follow exactly
    the run's float32 arithmetic, so a sample pushed through ``run.fields`` lands on
    its frame bit-for-bit.  Fields built in float64 by the caller are applied in
    float64.
    """
    if isinstance(fields, RegularizationRun):
        fields = fields.fields
    if upto is None:
        upto = len(fields)
    chosen = list(fields[:upto])
    out = np.asarray(points, dtype=np.float64)
    if not chosen:
        return out
    if any(f.device_targets64() is not None for f in chosen):
        for f in chosen:
            out = sample_points(f, out, clip=True)
        return out
    shape = out.shape
    flat = out.reshape(-1, 2)
    if len(flat) == 0:
        return out
    return D.to_host64(map_through_device(chosen, D.to_device(flat))).reshape(shape)


def map_through_device(fields, pts: torch.Tensor) -> torch.Tensor:
    """Float32 device points (n, 2) pushed through float32 device fields (sample +
    clip per field, the run's own move arithmetic); returns a new device tensor."""
    lib = D.require_cuda()
    n = pts.shape[0]
    a = pts.contiguous().clone()
    if n == 0 or not fields:
        return a
    bbuf = torch.empty_like(a)
    for f in fields:
        _lib.check(lib.inim_sample(D.ptr(f.device_targets()), f.k, D.ptr(a), D.ptr(bbuf), n, 1, None, D.stream()),
                   "map_through")
        a, bbuf = bbuf, a
    return a
