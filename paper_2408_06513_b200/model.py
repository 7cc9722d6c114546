"""Domain types of the drop-in, mirroring the reference's model.py (uncrowd model.py:27-244).

Coordinate convention (model.py:1-8): grids are 2^k x 2^k, row-major, ``values[j, i]``
with i = x (column), j = y (row); pixel (i, j) <-> texture coordinate 2^-k (i, j).

Difference from the reference: the array-valued members (density values, the eight
tables, field targets, run frames) live on the GPU and are materialised as float64
host arrays only when read, so a pipeline of drop-in calls never round-trips through
the host.  Reading them gives the same shapes and dtype (float64) the reference
returns.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .errors import CoordinateOutOfRange, InvalidParams, LabelLengthMismatch, NonFiniteCoordinate, OutOfRangeLevel


class ScatterDataset:
    """Ordered 2-D samples in the unit square (model.py:27-41): positions, optional
    labels, and ids (default 0..n-1, materialised on first access so that wrapping a
    large array costs nothing).  Immutable, like the reference's frozen dataclass."""

    __slots__ = ("positions", "labels", "_ids")

    def __init__(self, positions: np.ndarray, labels: Optional[np.ndarray] = None, ids: Optional[np.ndarray] = None):
        object.__setattr__(self, "positions", positions)
        object.__setattr__(self, "labels", labels)
        object.__setattr__(self, "_ids", ids)

    def __setattr__(self, name, value):
        raise AttributeError("ScatterDataset is immutable")

    @property
    def ids(self) -> np.ndarray:
        if self._ids is None:
            object.__setattr__(self, "_ids", np.arange(len(self.positions)))
        return self._ids

    @property
    def n(self) -> int:
        return len(self.positions)

    def __repr__(self) -> str:
        return f"ScatterDataset(n={self.n}, labels={'yes' if self.labels is not None else 'no'})"


class _DeviceBacked:
    """Host view of a device tensor, materialised (float64) on first access."""

    __slots__ = ()

    @staticmethod
    def _host(dev, cache: dict, key: str, shape=None):
        if key not in cache:
            from ._device import to_host64

            arr = to_host64(dev)
            cache[key] = arr.reshape(shape) if shape is not None else arr
        return cache[key]


class DensityTexture(_DeviceBacked):
    """Smoothed per-pixel density plus the background constant (model.py:44-56)."""

    __slots__ = ("_values", "_dev", "_cache", "k", "kernel_size", "background", "n")

    def __init__(self, values=None, k: int = 0, kernel_size: int = 0, background: float = 0.0, n: int = 0, *,
                 device_values=None):
        self._values = None if values is None else np.asarray(values, dtype=np.float64)
        self._dev = device_values
        self._cache: dict = {}
        self.k, self.kernel_size, self.background, self.n = int(k), int(kernel_size), float(background), int(n)

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            self._values = self._host(self._dev, self._cache, "values")
        return self._values

    @property
    def size(self) -> int:
        return 1 << self.k

    def device_values(self):
        """float32 (s, s) device tensor of the values (uploaded on first use)."""
        if self._dev is None:
            from ._device import to_device

            self._dev = to_device(self._values)
        return self._dev


_TABLE_NAMES = ("rect_tl", "rect_bl", "rect_br", "rect_tr", "wedge_up", "wedge_left", "wedge_down", "wedge_right")


class IntegralSet(_DeviceBacked):
    """The eight per-pixel integral tables of a texture (model.py:59-85).

    Order of ``tables()``: rect tl, bl, br, tr, then wedge up, left, down, right.
    Each family partitions the domain, so both quadruples sum to ``total``.
    """

    __slots__ = ("_dev", "_host_tables", "_cache", "total", "k")

    def __init__(self, rect_tl=None, rect_bl=None, rect_br=None, rect_tr=None, wedge_up=None, wedge_left=None,
                 wedge_down=None, wedge_right=None, total: float = 0.0, k: int = 0, *, device_tables=None):
        given = (rect_tl, rect_bl, rect_br, rect_tr, wedge_up, wedge_left, wedge_down, wedge_right)
        self._host_tables = None
        if device_tables is None:
            self._host_tables = tuple(np.asarray(t, dtype=np.float64) for t in given)
        self._dev = device_tables  # float32 (8, s, s)
        self._cache: dict = {}
        self.total = float(total)
        self.k = int(k)

    def _table(self, idx: int) -> np.ndarray:
        if self._host_tables is not None:
            return self._host_tables[idx]
        if "all" not in self._cache:
            self._cache["all"] = self._host(self._dev, self._cache, "_t8")
        return self._cache["all"][idx]

    rect_tl = property(lambda self: self._table(0))
    rect_bl = property(lambda self: self._table(1))
    rect_br = property(lambda self: self._table(2))
    rect_tr = property(lambda self: self._table(3))
    wedge_up = property(lambda self: self._table(4))
    wedge_left = property(lambda self: self._table(5))
    wedge_down = property(lambda self: self._table(6))
    wedge_right = property(lambda self: self._table(7))

    def tables(self):
        return tuple(self._table(i) for i in range(8))

    def device_tables(self):
        """float32 (8, s, s) device tensor (uploaded on first use)."""
        if self._dev is None:
            from ._device import to_device

            self._dev = to_device(np.stack(self._host_tables))
        return self._dev


class DeformationField(_DeviceBacked):
    """Per-pixel target coordinates of one deformation step (model.py:88-98)."""

    __slots__ = ("_targets", "_dev", "_dev64", "_cache", "k", "max_excursion")

    def __init__(self, targets=None, k: int = 0, max_excursion: float = 0.0, *, device_targets=None):
        self._targets = None if targets is None else np.asarray(targets, dtype=np.float64)
        self._dev = device_targets   # float32 (s, s, 2), produced by the device pipeline
        self._dev64 = None           # float64 copy of caller-provided targets
        self._cache: dict = {}
        self.k = int(k)
        self.max_excursion = float(max_excursion)

    @property
    def targets(self) -> np.ndarray:
        if self._targets is None:
            self._targets = self._host(self._dev, self._cache, "targets")
        return self._targets

    @property
    def size(self) -> int:
        return 1 << self.k

    def device_targets(self):
        """float32 (s, s, 2) device tensor."""
        if self._dev is None:
            from ._device import to_device

            self._dev = to_device(self._targets)
        return self._dev

    def device_targets64(self):
        """float64 device copy when the field was built on the host in float64, else None."""
        if self._dev is not None:
            return None
        if self._dev64 is None:
            from ._device import to_device
            import torch

            self._dev64 = to_device(self._targets, dtype=torch.float64)
        return self._dev64


_STOP_KINDS = ("fixed", "displacement", "time")


@dataclass(frozen=True)
class RegularizationParams:
    """Run parameters and their validation (model.py:104-132)."""

    k: int = 10
    kernel_size: int = 8
    iterations: int = 16
    stop: str = "fixed"
    epsilon: float = 1e-4
    time_budget: Optional[float] = None
    background: Optional[float] = None
    frame_cap: int = 64

    def validate(self) -> "RegularizationParams":
        checks = (
            (self.k >= 1, "k must be >= 1"),
            (self.kernel_size >= 1, "kernel_size must be >= 1"),
            (self.iterations >= 0, "iterations must be >= 0"),
            (self.stop in _STOP_KINDS, f"stop must be one of {_STOP_KINDS}"),
            (self.stop != "displacement" or self.epsilon > 0, "epsilon must be > 0"),
            (self.stop != "time" or (self.time_budget is not None and self.time_budget > 0),
             "time_budget must be > 0 for stop='time'"),
            (self.background is None or self.background > 0, "explicit background must be > 0"),
            (self.frame_cap >= 2, "frame_cap must be >= 2"),
        )
        for ok, msg in checks:
            if not ok:
                raise InvalidParams(msg)
        return self


class RegularizationRun:
    """Original dataset plus per-iteration frames, fields and wall times
    (model.py:135-180).

    Frames are kept as float32 device tensors under the reference's ``frame_cap``
    thinning policy (every other kept frame is dropped when the cap is exceeded);
    a dropped frame is recomputed on demand from the nearest kept predecessor with
    the same device iteration, which is deterministic, so the recomputed frame is
    bit-identical to the one the run produced.
    """

    def __init__(self, dataset: ScatterDataset, params: RegularizationParams, store_fields: bool = True):
        self.original = dataset
        self.params = params
        self.store_fields = store_fields
        self.fields: list = []
        self.metrics: list = []
        self._dev_frames: dict = {}      # t -> float32 (n, 2) device tensor (t >= 1)
        self._host_frames: dict = {0: dataset.positions}
        self._pending: dict = {}         # t -> (pinned host tensor, event): copy in flight
        self._stride = 1
        self.iterations = 0
        self.wall_times: list = []

    def _record(self, t: int, dev_positions):
        self._dev_frames[t] = dev_positions
        self.iterations = max(self.iterations, t)
        kept = {0, *self._dev_frames}
        if len(kept) > self.params.frame_cap:
            self._stride *= 2
            keep = {0, self.iterations} | {i for i in kept if i % self._stride == 0}
            for i in list(self._dev_frames):
                if i not in keep:
                    del self._dev_frames[i]
                    self._host_frames.pop(i, None)
                    self._pending.pop(i, None)

    def _prefetch(self, t: int):
        """Start the host copy of kept frame t now (the run's last frame): it overlaps
        the host-side bookkeeping, and frame(t) only waits for it."""
        from ._device import to_host64_async

        if t in self._dev_frames and t not in self._host_frames and t not in self._pending:
            self._pending[t] = to_host64_async(self._dev_frames[t])

    def _device_frame(self, t: int):
        from ._device import to_device

        if t == 0:
            return to_device(self.original.positions).reshape(-1, 2)
        return self._dev_frames[t]

    def frame(self, t: int) -> np.ndarray:
        """Positions after t iterations (t = 0 is the input layout)."""
        if not 0 <= t <= self.iterations:
            raise OutOfRangeLevel(f"frame {t} outside [0, {self.iterations}]")
        if t in self._host_frames:
            return self._host_frames[t]
        if t in self._pending:
            host, ev = self._pending.pop(t)
            ev.synchronize()
            self._host_frames[t] = host.numpy()
            return self._host_frames[t]
        from ._device import to_host64
        from .regularize import _device_iterate

        if t in self._dev_frames:
            arr = to_host64(self._dev_frames[t])
        else:
            base = max(i for i in (0, *self._dev_frames) if i <= t)
            pos = self._device_frame(base)
            for _ in range(base, t):
                pos, _ = _device_iterate(pos, self.params, with_field=False)
            arr = to_host64(pos)
        self._host_frames[t] = arr
        return arr

    @property
    def frames(self) -> list:
        return [self.frame(t) for t in range(self.iterations + 1)]


def unit_coordinates(k: int):
    """Per-pixel texture coordinates (X, Y), each (2^k, 2^k) (model.py:183-186)."""
    axis = np.arange(1 << k, dtype=np.float64) * (2.0 ** -k)
    return np.meshgrid(axis, axis, indexing="xy")


def pixel_of(x, y, k: int):
    """Pixel indices (i, j) containing (x, y); the right/bottom edge clamps into the
    last pixel (model.py:189-198).  Host index arithmetic for callers; the device
    splat applies the same rule internally."""
    size = 1 << k
    i = np.minimum(np.floor(np.asarray(x) * size), size - 1).astype(np.int64)
    j = np.minimum(np.floor(np.asarray(y) * size), size - 1).astype(np.int64)
    return i, j


def validate_dataset(raw, labels: Optional[Sequence] = None, normalize: bool = True) -> ScatterDataset:
    """Validate raw coordinate pairs into a ScatterDataset (model.py:201-244): finite
    check, optional per-axis min-max normalization (degenerate axis -> 0.5), label
    length check and integer relabelling."""
    pts = np.asarray(raw, dtype=np.float64)
    if pts.size == 0:
        pts = pts.reshape(0, 2)
    if pts.ndim != 2 or pts.shape[1] != 2:
        raise ValueError("expected an (n, 2) array of coordinate pairs")
    finite = np.isfinite(pts)
    if not finite.all():
        row = int(np.argwhere(~finite)[0][0])
        raise NonFiniteCoordinate(f"non-finite coordinate at row {row}")
    if len(pts) and normalize:
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        span = hi - lo
        scaled = np.empty_like(pts)
        for ax in (0, 1):
            scaled[:, ax] = 0.5 if span[ax] == 0.0 else (pts[:, ax] - lo[ax]) / span[ax]
        pts = scaled
    elif len(pts) and (pts.min() < 0.0 or pts.max() > 1.0):
        raise CoordinateOutOfRange("coordinates outside [0,1]^2; pass normalize=True to rescale")
    lab = None
    if labels is not None:
        if len(labels) != len(pts):
            raise LabelLengthMismatch(f"{len(labels)} labels for {len(pts)} samples")
        lab = np.asarray(labels)
        if lab.dtype.kind not in "iu":
            _u, lab = np.unique(lab, return_inverse=True)
        lab = lab.astype(np.int64)
    return ScatterDataset(positions=pts, labels=lab)


def elapsed_ms(start: float) -> float:
    return (time.perf_counter() - start) * 1e3
