"""Deformation map, field and bilinear sampling on the GPU (drop-in for uncrowd
mapping.py:24-251).

build_field       -> inim_field_from_tables (per-pixel Eq. (map) minus the flat response)
sample_field      -> inim_sample_f64 / inim_sample_t64 (bilinear, one-sided last cell)
anchors / raw_map / corrected_map -> inim_map_points (query points, float64)
flat_response     -> inim_flat_response_f64 (closed-form region counts), cached per k
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import SingularMass
from .model import DeformationField, IntegralSet


@dataclass(frozen=True)
class AnchorSet:
    """Exit points of the four diagonal rays through (x, y) (mapping.py:24-33)."""

    down_right: np.ndarray
    up_right: np.ndarray
    up_left: np.ndarray
    down_left: np.ndarray


def _points(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    x, y = np.broadcast_arrays(x, y)
    return x.shape, np.ascontiguousarray(x).ravel(), np.ascontiguousarray(y).ravel()


def _map_points(x, y, mode: int, tables: IntegralSet = None, defect64=None):
    lib = D.require_cuda()
    shape, xs, ys = _points(x, y)
    n = xs.size
    width = 8 if mode == 0 else 2
    xd = torch.from_numpy(xs).to(D.device())
    yd = torch.from_numpy(ys).to(D.device())
    out = torch.empty((max(n, 1), width), dtype=torch.float64, device=D.device())
    t8 = tables.device_tables() if tables is not None else None
    tot = torch.tensor([tables.total], dtype=torch.float64, device=D.device()) if tables is not None else None
    k = tables.k if tables is not None else 0
    _lib.check(lib.inim_map_points(D.ptr(t8), k, D.ptr(tot), D.ptr(defect64), D.ptr(xd), D.ptr(yd), n, mode,
                                   D.ptr(out), D.stream()), "map_points")
    return shape, out[:n].cpu().numpy()


def anchors(x, y) -> AnchorSet:
    """The four diagonal exit points for coordinates in [0,1]^2 (mapping.py:55-61)."""
    shape, o = _map_points(x, y, 0)
    q = [o[:, 2 * c:2 * c + 2].reshape(shape + (2,)) for c in range(4)]
    return AnchorSet(down_right=q[0], up_right=q[1], up_left=q[2], down_left=q[3])


def raw_map(x, y, tables: IntegralSet) -> np.ndarray:
    """Weighted anchor combination at the pixel containing (x, y) (mapping.py:80-101)."""
    if not tables.total > 0.0:
        raise SingularMass("total texture mass must be > 0")
    shape, o = _map_points(x, y, 1, tables)
    return o.reshape(shape + (2,))


class _FlatResponseCache:
    """Raw-map response of a flat texture, built once per resolution (mapping.py:104-129).

    Built on the device from the closed-form region pixel counts of a constant texture
    (exact integers) in float64; ``builds`` counts constructions exactly like the
    reference.  The fused device iteration evaluates the same closed form in registers
    instead of reading this array.
    """

    def __init__(self):
        self._cache: dict = {}
        self.builds = 0

    def clear(self):
        self._cache.clear()
        self.builds = 0

    def _entry(self, k: int):
        """The cache slot of k; creating it counts as one build (the arrays themselves
        are materialised on first use: at k = 15 each is 16 GiB)."""
        if k not in self._cache:
            D.check_grid(k)
            self._cache[k] = {"host": None, "dev64": None}
            self.builds += 1
        return self._cache[k]

    def get(self, k: int) -> np.ndarray:
        e = self._entry(k)
        if e["host"] is None:
            e["host"] = self.device64(k).cpu().numpy()
        return e["host"]

    def is_flat(self, k: int, defect) -> bool:
        """True when `defect` is this cache's array for k (then the closed form is used)."""
        e = self._cache.get(k)
        return e is not None and e["host"] is not None and defect is e["host"]

    def device64(self, k: int):
        e = self._entry(k)
        if e["dev64"] is None:
            lib = D.require_cuda()
            s = 1 << k
            dev64 = torch.empty((s, s, 2), dtype=torch.float64, device=D.device())
            _lib.check(lib.inim_flat_response_f64(k, D.ptr(dev64), D.stream()), "flat_response")
            e["dev64"] = dev64
        return e["dev64"]

    def touch(self, k: int) -> None:
        """Register the build of k without materialising it (regularize.run)."""
        self._entry(k)


flat_response = _FlatResponseCache()


def _defect_device(k: int, defect, dtype):
    """Device copy of an explicit defect array, or None for the flat response."""
    if defect is None or flat_response.is_flat(k, defect):
        return None
    return D.to_device(np.asarray(defect, dtype=np.float64), dtype=dtype)


def corrected_map(x, y, tables: IntegralSet, defect) -> np.ndarray:
    """clip((x, y) + raw(x, y) - defect[containing pixel]) (mapping.py:132-143)."""
    if not tables.total > 0.0:
        raise SingularMass("total texture mass must be > 0")
    d64 = _defect_device(tables.k, defect, torch.float64)
    if d64 is None:
        d64 = flat_response.device64(tables.k)
    shape, o = _map_points(x, y, 2, tables, d64)
    return o.reshape(shape + (2,))


def build_field(tables: IntegralSet, defect: np.ndarray = None) -> DeformationField:
    """Corrected targets at every pixel coordinate 2^-k (i, j), clipped, with the
    pre-clip excursion (mapping.py:194-204)."""
    if defect is None:
        defect = flat_response.get(tables.k)
    if not tables.total > 0.0:
        raise SingularMass("total texture mass must be > 0")
    lib = D.require_cuda()
    k = tables.k
    s = 1 << k
    dev_def = _defect_device(k, defect, torch.float32)
    targets = torch.empty((s, s, 2), dtype=torch.float32, device=D.device())
    exc = torch.zeros(1, dtype=torch.float32, device=D.device())
    tot = torch.tensor([tables.total], dtype=torch.float64, device=D.device())
    _lib.check(lib.inim_field_from_tables(D.ptr(tables.device_tables()), k, D.ptr(tot), D.ptr(dev_def),
                                          D.ptr(targets), D.ptr(exc), D.stream()), "build_field")
    return DeformationField(k=k, max_excursion=float(exc.item()), device_targets=targets)


def sample_points(field: DeformationField, points, clip: bool) -> np.ndarray:
    """Bilinear field evaluation at float64 points [+ clip to [0,1]] on the device."""
    lib = D.require_cuda()
    pts = np.asarray(points, dtype=np.float64)
    flat = np.ascontiguousarray(pts.reshape(-1, 2))
    n = len(flat)
    if n == 0:
        return pts.copy()
    src = torch.from_numpy(flat).to(D.device())
    out = torch.empty_like(src)
    t64 = field.device_targets64()
    if t64 is not None:
        rc = lib.inim_sample_t64(D.ptr(t64), field.k, D.ptr(src), D.ptr(out), n, int(clip), D.stream())
    else:
        rc = lib.inim_sample_f64(D.ptr(field.device_targets()), field.k, D.ptr(src), D.ptr(out), n, int(clip),
                                 D.stream())
    _lib.check(rc, "sample_field")
    return out.cpu().numpy().reshape(pts.shape)


def sample_field(field: DeformationField, points: np.ndarray) -> np.ndarray:
    """Bilinear blend of the four pixel targets around each point (mapping.py:235-246)."""
    return sample_points(field, points, clip=False)


def interpolate(field: DeformationField, point) -> np.ndarray:
    """Single-point convenience wrapper around sample_field (mapping.py:249-251)."""
    return sample_field(field, np.asarray(point, dtype=np.float64))
