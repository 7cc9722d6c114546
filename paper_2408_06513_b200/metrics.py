"""Layout-quality metrics on the GPU (drop-in for uncrowd metrics.py:1-168).

The device produces integers only -- occupied pixels and the sum of squared 4x4-bin
counts off a frame's splat counts (inim_frame_stats), the trustworthiness penalty sum
(inim_trust_penalty) and the preserved-pair count (inim_order_pairs) -- and the host
turns them into the reference's floats:

  binned_stddev   sqrt(var), var = (B*sum c^2 - (sum c)^2) / B^2 from exact integers
                  (the reference's numpy std of the same integer bin counts, metrics.py:59)
  overplotting    (n - occupied) / n                       (metrics.py:71, exact)
  trustworthiness 1 - penalties / (n*nn*(2n - 3nn - 1)/2)  (metrics.py:109-113, exact)
  ordering        preserved / (n*(n-1)/2)                  (metrics.py:143-144, exact)

The fixed-seed subsample of the pair metrics (PCG64 seed 1789, metrics.py:15-16,
132-134, 162-166) is drawn on the host with numpy's own generator, so the same rows are
picked; it is index bookkeeping, not arithmetic.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import EmptyDataset, TooFewSamples

BIN_PIXELS = 4  # occupancy statistics use 4x4-pixel bins
_SUBSAMPLE_CAP = 4096
_SUBSAMPLE_SEED = 1789


@dataclass(frozen=True)
class MetricRecord:
    """One frame's metrics (metrics.py:19-43)."""

    iteration: int
    binned_stddev: float
    overplotting: float
    trustworthiness: Optional[float]
    ordering: Optional[float]
    wall_ms: float

    def to_json_line(self) -> str:
        # fixed key order, wall time excluded: identical runs export identical bytes
        return json.dumps({
            "iteration": self.iteration,
            "binned_stddev": self.binned_stddev,
            "overplotting": self.overplotting,
            "trustworthiness": self.trustworthiness,
            "ordering": self.ordering,
        })

    @staticmethod
    def from_json_line(line: str) -> "MetricRecord":
        d = json.loads(line)
        d.setdefault("wall_ms", 0.0)
        return MetricRecord(**d)


# ------------------------------------------------------------------ integer -> float
def stddev_from_stats(sum_sq: int, total: int, k: int) -> float:
    """Population std of the 4x4-bin counts from their exact integer moments."""
    nb = ((1 << k) // BIN_PIXELS) ** 2
    return math.sqrt((nb * int(sum_sq) - int(total) * int(total)) / (nb * nb))


def overplotting_from_stats(occupied: int, n: int) -> float:
    return (n - int(occupied)) / n


def trust_from_penalty(penalty: int, n: int, n_neighbors: int) -> float:
    total = float(penalty)
    if total == 0.0:
        return 1.0
    norm = n * n_neighbors * (2 * n - 3 * n_neighbors - 1) / 2.0
    return 1.0 - total / norm


def ordering_from_pairs(preserved: int, n: int) -> float:
    return int(preserved) / (n * (n - 1) / 2)


def subsample_rows(n: int, cap: int = _SUBSAMPLE_CAP) -> Optional[np.ndarray]:
    """Rows of the fixed-seed subsample (metrics.py:132-134, 162-165); None if n <= cap."""
    if n <= cap:
        return None
    rng = np.random.Generator(np.random.PCG64(_SUBSAMPLE_SEED))
    return rng.choice(n, size=cap, replace=False)


# ------------------------------------------------------------------------ device legs
def _points_f64(a) -> torch.Tensor:
    """(n, 2) float64 device tensor (device float32 frames widen exactly)."""
    D.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=D.device(), dtype=torch.float64).reshape(-1, 2).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 2)).to(D.device())


def frame_stats(positions, k: int) -> tuple[int, int, int]:
    """(occupied pixels, sum of squared 4x4-bin counts, n) of a layout: one splat
    (bit-exact pixel_of binning) and one reduction on the device."""
    lib = D.require_cuda()
    s = 1 << k
    pts = _points_f64(positions)
    n = pts.shape[0]
    if n and (not bool(torch.isfinite(pts).all()) or bool((pts < 0).any())):
        raise ValueError("positions must be finite and non-negative")
    counts = torch.zeros((s, s), dtype=torch.int32, device=D.device())
    out = torch.zeros(3, dtype=torch.int64, device=D.device())
    if n:
        _lib.check(lib.inim_splat(D.ptr(pts), 1, n, k, D.ptr(counts), D.stream()), "splat")
    _lib.check(lib.inim_frame_stats(D.ptr(counts), k, D.ptr(out), D.stream()), "frame_stats")
    occ, sq, tot = (int(v) for v in out.cpu().tolist())
    return occ, sq, tot


def _trust_penalty(orig: torch.Tensor, moved: torch.Tensor, n_neighbors: int) -> int:
    lib = D.require_cuda()
    out = torch.zeros(1, dtype=torch.int64, device=D.device())
    _lib.check(lib.inim_trust_penalty(D.ptr(orig), D.ptr(moved), orig.shape[0], int(n_neighbors), D.ptr(out),
                                      D.stream()), "trustworthiness")
    return int(out.item())


def _order_pairs(orig: torch.Tensor, moved: torch.Tensor) -> int:
    lib = D.require_cuda()
    out = torch.zeros(1, dtype=torch.int64, device=D.device())
    _lib.check(lib.inim_order_pairs(D.ptr(orig), D.ptr(moved), orig.shape[0], D.ptr(out), D.stream()),
               "orthogonal_ordering")
    return int(out.item())


# ----------------------------------------------------------------------- public API
def binned_stddev(positions, k: int) -> float:
    """Population standard deviation of per-bin sample counts, 4x4-pixel bins
    (metrics.py:46-59)."""
    if k < 2:
        raise ValueError("k must be >= 2 so 4x4-pixel bins tile the grid")
    if len(positions) == 0:
        return 0.0
    _occ, sq, tot = frame_stats(positions, k)
    return stddev_from_stats(sq, tot, k)


def overplotting(positions, k: int) -> float:
    """(n - occupied pixels) / n (metrics.py:62-71)."""
    n = len(positions)
    if n == 0:
        raise EmptyDataset("overplotting needs at least one sample")
    occ, _sq, _tot = frame_stats(positions, k)
    return overplotting_from_stats(occ, n)


def trustworthiness(original, deformed, n_neighbors: int = 10) -> float:
    """Rank-based neighbourhood preservation in [0, 1] (metrics.py:74-113)."""
    original = np.asarray(original, dtype=np.float64) if not isinstance(original, torch.Tensor) else original
    deformed = np.asarray(deformed, dtype=np.float64) if not isinstance(deformed, torch.Tensor) else deformed
    n = len(original)
    if len(deformed) != n:
        raise ValueError("arrays must have the same length")
    if n <= n_neighbors:
        raise TooFewSamples(f"need more than {n_neighbors} samples")
    pen = _trust_penalty(_points_f64(original), _points_f64(deformed), n_neighbors)
    return trust_from_penalty(pen, n, n_neighbors)


def orthogonal_ordering(original, deformed, sample_cap: int = _SUBSAMPLE_CAP) -> float:
    """Fraction of sample pairs keeping both their x-order and y-order signs, on a
    fixed-seed subsample above `sample_cap` (metrics.py:116-144)."""
    original = np.asarray(original, dtype=np.float64) if not isinstance(original, torch.Tensor) else original
    deformed = np.asarray(deformed, dtype=np.float64) if not isinstance(deformed, torch.Tensor) else deformed
    n = len(original)
    if len(deformed) != n:
        raise ValueError("arrays must have the same length")
    if n < 2:
        return 1.0
    o, m = _points_f64(original), _points_f64(deformed)
    rows = subsample_rows(n, sample_cap)
    if rows is not None:
        idx = torch.from_numpy(rows).to(D.device())
        o, m, n = o[idx].contiguous(), m[idx].contiguous(), sample_cap
    return ordering_from_pairs(_order_pairs(o, m), n)


def record_for_frame(iteration: int, original, positions, k: int, wall_ms: float, full: bool = False,
                     n_neighbors: int = 10) -> MetricRecord:
    """Metric record for one run frame (metrics.py:147-168); neighbourhood metrics only
    in full mode, on the fixed-seed subsample above 4096 samples."""
    trust = order = None
    n = len(positions)
    if full and n > n_neighbors:
        o, m = _points_f64(original), _points_f64(positions)
        rows = subsample_rows(len(o))
        if rows is not None:
            idx = torch.from_numpy(rows).to(D.device())
            o, m = o[idx].contiguous(), m[idx].contiguous()
        trust = trustworthiness(o, m, n_neighbors=n_neighbors)
        order = orthogonal_ordering(o, m)
    if k < 2:  # binned_stddev's own check (metrics.py:52-53)
        raise ValueError("k must be >= 2 so 4x4-pixel bins tile the grid")
    if n:
        occ, sq, tot = frame_stats(positions, k)
        bsd, ovp = stddev_from_stats(sq, tot, k), overplotting_from_stats(occ, n)
    else:
        bsd, ovp = 0.0, 0.0
    return MetricRecord(iteration=iteration, binned_stddev=bsd, overplotting=ovp, trustworthiness=trust,
                        ordering=order, wall_ms=wall_ms)


class RunMetrics:
    """Device buffers of the per-frame metrics inside ``run`` (inim_run_metrics): the
    subsample of frame 0 is uploaded once; each chunk's integer statistics come back in
    one small copy."""

    def __init__(self, dataset_positions: np.ndarray, k: int, chunk: int, full: bool, n_neighbors: int):
        dev = D.device()
        self.k = k
        self.n = len(dataset_positions)
        self.n_neighbors = int(n_neighbors)
        self.fstats = torch.zeros((chunk, 3), dtype=torch.int64, device=dev)
        self.full = bool(full and self.n > n_neighbors)
        self.orig_sub = self.pick = self.moved_sub = self.nbstats = None
        self.n_sub = 0
        if self.full:
            rows = subsample_rows(self.n)
            base = np.ascontiguousarray(dataset_positions, dtype=np.float64).reshape(-1, 2)
            sub = base if rows is None else base[rows]
            self.n_sub = len(sub)
            if self.n_sub <= self.n_neighbors:
                raise TooFewSamples(f"need more than {self.n_neighbors} samples")
            self.orig_sub = torch.from_numpy(np.ascontiguousarray(sub)).to(dev)
            self.pick = None if rows is None else torch.from_numpy(rows.astype(np.int64)).to(dev)
            self.moved_sub = torch.empty_like(self.orig_sub)
            self.nbstats = torch.zeros((chunk, 2), dtype=torch.int64, device=dev)

    def args(self):
        return (D.ptr(self.fstats), D.ptr(self.orig_sub), D.ptr(self.pick), self.n_sub, self.n_neighbors,
                D.ptr(self.moved_sub), D.ptr(self.nbstats))

    def records(self, first_iteration: int, executed: int, wall_ms: float) -> list:
        if executed <= 0:
            return []
        fs = self.fstats[:executed].cpu().tolist()
        nb = self.nbstats[:executed].cpu().tolist() if self.full else None
        out = []
        for t in range(executed):
            occ, sq, tot = fs[t]
            trust = order = None
            if nb is not None:
                trust = trust_from_penalty(nb[t][0], self.n_sub, self.n_neighbors)
                order = ordering_from_pairs(nb[t][1], self.n_sub)
            out.append(MetricRecord(iteration=first_iteration + t, binned_stddev=stddev_from_stats(sq, tot, self.k),
                                    overplotting=overplotting_from_stats(occ, self.n) if self.n else 0.0,
                                    trustworthiness=trust, ordering=order, wall_ms=wall_ms))
        return out
