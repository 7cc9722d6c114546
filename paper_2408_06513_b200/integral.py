"""The eight integral tables on the GPU (drop-in for uncrowd integral.py:180-247).

build_integral_set runs the single-write-pass pipeline of csrc/integral.cu
(reduce -> float64 carry scan -> write).  The staged functions the reference also
exports (column_integrals, classical_rects, triangle_integrals, tilted_wedges) run as
float64-accumulated line scans on the device.

``scan_counter`` keeps the reference's observable contract (integral.py:26-40): every
staged scan adds k doubling steps, exactly as the reference's doubling scans do, even
though the device scans are single-pass.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as D
from . import _lib
from .model import DensityTexture, IntegralSet


class _StepCounter:
    """Doubling-step counter; tests assert k steps per scan per stage."""

    def __init__(self):
        self.steps = 0

    def reset(self):
        self.steps = 0


scan_counter = _StepCounter()


def _count_steps(size: int, scans: int = 1):
    scan_counter.steps += scans * max(0, int(size).bit_length() - 1)


@dataclass(frozen=True)
class ColumnIntegrals:
    """Per-pixel column sums: rows <= j (upper) and rows > j (lower)."""

    upper: np.ndarray
    lower: np.ndarray
    _dev: tuple = field(default=None, repr=False, compare=False)

    def device(self):
        if self._dev is None:
            object.__setattr__(self, "_dev", (D.to_device(self.upper), D.to_device(self.lower)))
        return self._dev


@dataclass(frozen=True)
class TriangleIntegrals:
    """Column integrals accumulated along the four diagonal directions."""

    up_left: np.ndarray
    up_right: np.ndarray
    down_left: np.ndarray
    down_right: np.ndarray
    _dev: tuple = field(default=None, repr=False, compare=False)

    def device(self):
        if self._dev is None:
            object.__setattr__(self, "_dev", tuple(D.to_device(t) for t in
                                                   (self.up_left, self.up_right, self.down_left, self.down_right)))
        return self._dev


def _texture_k(values) -> int:
    shape = values.shape
    if len(shape) != 2 or shape[0] != shape[1] or shape[0] < 1 or shape[0] & (shape[0] - 1):
        raise ValueError("texture must be square with a power-of-two side")
    return int(shape[0]).bit_length() - 1


def _scan(src: torch.Tensor, k: int, dj: int, di: int, exclusive: int) -> torch.Tensor:
    lib = D.require_cuda()
    out = torch.empty_like(src)
    _lib.check(lib.inim_line_scan(D.ptr(src), D.ptr(out), k, dj, di, exclusive, D.stream()), "line_scan")
    return out


def column_integrals(d) -> ColumnIntegrals:
    """Inclusive column prefix (upper) and strict column suffix (lower) (integral.py:180-186)."""
    values = np.asarray(d, dtype=np.float64)
    k = _texture_k(values)
    lib = D.require_cuda()
    src = D.to_device(values)
    up = torch.empty_like(src)
    lo = torch.empty_like(src)
    _lib.check(lib.inim_column_integrals(D.ptr(src), k, D.ptr(up), D.ptr(lo), D.stream()), "column_integrals")
    _count_steps(values.shape[0], 2)
    return ColumnIntegrals(upper=D.to_host64(up), lower=D.to_host64(lo), _dev=(up, lo))


def classical_rects(cols: ColumnIntegrals):
    """Corner rectangles (tl, bl, br, tr) from the column integrals (integral.py:189-200)."""
    up, lo = cols.device()
    k = _texture_k(cols.upper)
    tl = _scan(up, k, 0, 1, 0)
    bl = _scan(lo, k, 0, 1, 0)
    tr = _scan(up, k, 0, -1, 1)
    br = _scan(lo, k, 0, -1, 1)
    _count_steps(cols.upper.shape[1], 4)
    return tuple(D.to_host64(t) for t in (tl, bl, br, tr))


def triangle_integrals(cols: ColumnIntegrals) -> TriangleIntegrals:
    """Diagonal chains of upper toward up-left/up-right, of lower toward down-left/
    down-right (integral.py:203-209)."""
    up, lo = cols.device()
    k = _texture_k(cols.upper)
    ul = _scan(up, k, 1, 1, 0)
    ur = _scan(up, k, 1, -1, 0)
    dl = _scan(lo, k, -1, 1, 0)
    dr = _scan(lo, k, -1, -1, 0)
    _count_steps(cols.upper.shape[0], 4)
    return TriangleIntegrals(*(D.to_host64(t) for t in (ul, ur, dl, dr)), _dev=(ul, ur, dl, dr))


def tilted_wedges(tri: TriangleIntegrals, cols: ColumnIntegrals):
    """Wedges (up, left, down, right) by triangle arithmetic (integral.py:212-228)."""
    lib = D.require_cuda()
    ul, ur, dl, dr = tri.device()
    up, lo = cols.device()
    k = _texture_k(cols.upper)
    s = 1 << k
    out = torch.empty((4, s, s), dtype=torch.float32, device=D.device())
    scratch = torch.empty(2 * s, dtype=torch.float64, device=D.device())
    _lib.check(lib.inim_tilted_wedges(D.ptr(ul), D.ptr(ur), D.ptr(dl), D.ptr(dr), D.ptr(up), D.ptr(lo), k,
                                      D.ptr(scratch), D.ptr(out), D.stream()), "tilted_wedges")
    _count_steps(s, 2)
    host = D.to_host64(out)
    return host[0], host[1], host[2], host[3]


def build_integral_set(d) -> IntegralSet:
    """All eight tables plus the total mass (integral.py:231-247).

    Accepts a DensityTexture (its device values are used directly) or a square
    power-of-two array.  Tables are float32 on the device, read back as float64.
    """
    lib = D.require_cuda()
    if isinstance(d, DensityTexture):
        k = d.k
        src = d.device_values()
    else:
        values = np.asarray(d, dtype=np.float64)
        k = _texture_k(values)
        src = D.to_device(values)
    s = 1 << k
    tables = torch.empty((8, s, s), dtype=torch.float32, device=D.device())
    total = torch.empty(1, dtype=torch.float64, device=D.device())
    ws = D.workspace(k)
    _lib.check(lib.inim_integral_set(D.ptr(src), k, D.ptr(tables), D.ptr(total), D.ptr(ws), D.stream()),
               "build_integral_set")
    # the reference's staged scans: 2k + 4k + 4k + 2k doubling steps
    _count_steps(s, 12)
    return IntegralSet(total=float(total.item()), k=k, device_tables=tables)
