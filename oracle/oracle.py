"""ctypes front end of the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Wraps ``oracle/liboracle.so`` (built from ``inim_oracle.c`` by ``oracle/Makefile``), a
float64 restatement of the reference hot path (``uncrowd``: density.py, integral.py,
mapping.py, regularize.py).  Every function below names the reference symbol it
restates.  Only tests, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg import this module; the product package never does.

Pinned against golden vectors recorded from the real reference
(tests/golden/make_golden.py -> tests/golden/*.npz; checked by
tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def build(force: bool = False) -> Path:
    """Compile the C restatement (``make -C oracle``)."""
    src = _HERE / "inim_oracle.c"
    if force or not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.orc_set_threads.argtypes = [ctypes.c_int]
        L.orc_set_threads.restype = ctypes.c_int
        L.orc_accumulate.argtypes = [_dp, _i64, ctypes.c_int, _dp]
        L.orc_smoothing_kernel.argtypes = [ctypes.c_int, _dp]
        L.orc_gaussian_smooth.argtypes = [_dp, _i64, ctypes.c_int, _dp]
        L.orc_build_density.argtypes = [_dp, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_double, _dp, _dp]
        L.orc_column_integrals.argtypes = [_dp, _i64, _dp, _dp]
        L.orc_build_integral_set.argtypes = [_dp, _i64, _dp, _dp]
        L.orc_raw_targets_per_pixel.argtypes = [_dp, ctypes.c_double, ctypes.c_int, _dp]
        L.orc_flat_response.argtypes = [ctypes.c_int, _dp]
        L.orc_build_field.argtypes = [_dp, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp]
        L.orc_sample_field.argtypes = [_dp, ctypes.c_int, _dp, _i64, _dp]
        L.orc_iterate_once.argtypes = [_dp, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       _dp, _dp, _dp, _dp, _dp]
        L.orc_sum.argtypes = [_dp, _i64]
        L.orc_sum.restype = ctypes.c_double
        _lib = L
        threads = int(os.environ.get("INIM_ORACLE_THREADS", "0"))
        if threads > 0:
            L.orc_set_threads(threads)
    return _lib


def set_threads(n: int) -> int:
    return lib().orc_set_threads(int(n))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(rc: int, what: str):
    if rc == 1:
        raise ValueError(f"oracle {what}: invalid argument")
    if rc == 2:
        raise MemoryError(f"oracle {what}: out of memory")
    if rc == 3:
        raise ValueError(f"oracle {what}: total texture mass must be > 0")
    if rc:
        raise RuntimeError(f"oracle {what}: error {rc}")


def accumulate(positions, k: int) -> np.ndarray:
    """density.accumulate (density.py:14-27)."""
    pos = _f64(positions).reshape(-1, 2)
    s = 1 << k
    grid = np.empty((s, s))
    _check(lib().orc_accumulate(_p(pos), len(pos), k, _p(grid)), "accumulate")
    return grid


def smoothing_kernel(kernel_size: int) -> np.ndarray:
    """density.smoothing_kernel (density.py:30-37)."""
    w = np.empty(6 * kernel_size + 1)
    _check(lib().orc_smoothing_kernel(kernel_size, _p(w)), "smoothing_kernel")
    return w


def gaussian_smooth(grid, kernel_size: int) -> np.ndarray:
    """density.gaussian_smooth (density.py:40-51)."""
    g = _f64(grid)
    out = np.empty_like(g)
    _check(lib().orc_gaussian_smooth(_p(g), g.shape[0], kernel_size, _p(out)), "gaussian_smooth")
    return out


def build_density(positions, k: int, kernel_size: int, background=None):
    """density.build_density (density.py:54-78) -> (values, background)."""
    pos = _f64(positions).reshape(-1, 2)
    s = 1 << k
    values = np.empty((s, s))
    bg = ctypes.c_double(0.0)
    b = -1.0 if background is None else float(background)
    _check(lib().orc_build_density(_p(pos), len(pos), k, kernel_size, b, _p(values), ctypes.byref(bg)),
           "build_density")
    return values, bg.value


def column_integrals(d):
    """integral.column_integrals (integral.py:180-186) -> (upper, lower)."""
    d = _f64(d)
    upper = np.empty_like(d)
    lower = np.empty_like(d)
    _check(lib().orc_column_integrals(_p(d), d.shape[0], _p(upper), _p(lower)), "column_integrals")
    return upper, lower


def build_integral_set(d):
    """integral.build_integral_set (integral.py:231-247) -> (tables[8,s,s], total)."""
    d = _f64(d)
    s = d.shape[0]
    if d.ndim != 2 or d.shape[1] != s or s & (s - 1):
        raise ValueError("texture must be square with a power-of-two side")
    t8 = np.empty((8, s, s))
    total = ctypes.c_double(0.0)
    _check(lib().orc_build_integral_set(_p(d), s, _p(t8), ctypes.byref(total)), "build_integral_set")
    return t8, total.value


def raw_targets_per_pixel(tables8, total: float, k: int) -> np.ndarray:
    """mapping._raw_targets_per_pixel (mapping.py:181-191)."""
    t8 = _f64(tables8)
    s = 1 << k
    out = np.empty((s, s, 2))
    _check(lib().orc_raw_targets_per_pixel(_p(t8), float(total), k, _p(out)), "raw_targets")
    return out


def flat_response(k: int) -> np.ndarray:
    """mapping.flat_response.get(k) (mapping.py:120-126)."""
    s = 1 << k
    out = np.empty((s, s, 2))
    _check(lib().orc_flat_response(k, _p(out)), "flat_response")
    return out


def build_field(tables8, total: float, k: int, defect=None):
    """mapping.build_field (mapping.py:194-204) -> (targets, max_excursion)."""
    t8 = _f64(tables8)
    if defect is None:
        defect = flat_response(k)
    defect = _f64(defect)
    s = 1 << k
    out = np.empty((s, s, 2))
    exc = ctypes.c_double(0.0)
    _check(lib().orc_build_field(_p(t8), float(total), k, _p(defect), _p(out), ctypes.byref(exc)), "build_field")
    return out, exc.value


def sample_field(targets, points) -> np.ndarray:
    """mapping.sample_field (mapping.py:207-246)."""
    t = _f64(targets)
    k = int(t.shape[0]).bit_length() - 1
    pts = _f64(points)
    flat = pts.reshape(-1, 2)
    out = np.empty_like(flat)
    _check(lib().orc_sample_field(_p(t), k, _p(flat), len(flat), _p(out)), "sample_field")
    return out.reshape(pts.shape)


def iterate_once(positions, k: int, kernel_size: int, background=None, defect=None,
                 want_field: bool = False, want_density: bool = False):
    """regularize.iterate_once (regularize.py:25-37) -> new positions [, field, density]."""
    pos = _f64(positions).reshape(-1, 2)
    s = 1 << k
    new = np.empty_like(pos)
    field = np.empty((s, s, 2)) if want_field else None
    dens = np.empty((s, s)) if want_density else None
    if defect is not None:
        defect = _f64(defect)
    b = -1.0 if background is None else float(background)
    exc = ctypes.c_double(0.0)
    null = ctypes.cast(None, _dp)
    _check(lib().orc_iterate_once(_p(pos), len(pos), k, kernel_size, b,
                                  _p(defect) if defect is not None else null, _p(new),
                                  _p(field) if field is not None else null,
                                  _p(dens) if dens is not None else null, ctypes.byref(exc)),
           "iterate_once")
    if want_field or want_density:
        return new, field, dens
    return new


def run_positions(positions, k: int, kernel_size: int, iterations: int, background=None,
                  stop: str = "fixed", epsilon: float = 1e-4):
    """regularize.run (regularize.py:40-80) restricted to the numeric path: returns the
    list of frames [frame0, frame1, ...] (no metrics, no thinning)."""
    pos = _f64(positions).reshape(-1, 2)
    defect = flat_response(k)
    frames = [pos]
    for _t in range(iterations):
        new = iterate_once(pos, k, kernel_size, background, defect)
        frames.append(new)
        disp = float(np.abs(new - pos).max()) if len(pos) else 0.0
        pos = new
        if stop == "displacement" and disp < epsilon:
            break
    return frames


def total(values) -> float:
    """float(values.sum()) restated with numpy's pairwise summation (integral.py:246)."""
    v = _f64(values).ravel()
    return lib().orc_sum(_p(v), len(v))


# ------------------------------------------------------------------ layout metrics
_SUBSAMPLE_CAP = 4096
_SUBSAMPLE_SEED = 1789


def _i64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _metric_lib():
    L = lib()
    if not getattr(L, "_metrics_typed", False):
        ip = ctypes.POINTER(ctypes.c_int64)
        L.orc_frame_stats.argtypes = [_dp, _i64, ctypes.c_int, ip]
        L.orc_trust_penalty.argtypes = [_dp, _dp, _i64, ctypes.c_int, ip]
        L.orc_order_pairs.argtypes = [_dp, _dp, _i64, ip]
        L._metrics_typed = True
    return L


def frame_stats(positions, k: int):
    """(occupied pixels, sum of squared 4x4-bin counts, n) (metrics.py:46-71)."""
    pos = _f64(positions).reshape(-1, 2)
    out = np.zeros(3, dtype=np.int64)
    _check(_metric_lib().orc_frame_stats(_p(pos), len(pos), k, _i64p(out)), "frame_stats")
    return tuple(int(v) for v in out)


def binned_stddev(positions, k: int) -> float:
    """metrics.binned_stddev (metrics.py:46-59): population std of the 4x4-bin counts,
    from their exact integer moments (var = (B sum c^2 - n^2) / B^2, correctly rounded)."""
    if k < 2:
        raise ValueError("k must be >= 2 so 4x4-pixel bins tile the grid")
    if len(positions) == 0:
        return 0.0
    _occ, sq, n = frame_stats(positions, k)
    nb = ((1 << k) // 4) ** 2
    return float(np.sqrt((nb * sq - n * n) / (nb * nb)))


def overplotting(positions, k: int) -> float:
    """metrics.overplotting (metrics.py:62-71)."""
    n = len(positions)
    if n == 0:
        raise ValueError("overplotting needs at least one sample")
    occ, _sq, _n = frame_stats(positions, k)
    return (n - occ) / n


def trust_penalty(original, deformed, n_neighbors: int = 10) -> int:
    o, m = _f64(original).reshape(-1, 2), _f64(deformed).reshape(-1, 2)
    out = np.zeros(1, dtype=np.int64)
    _check(_metric_lib().orc_trust_penalty(_p(o), _p(m), len(o), int(n_neighbors), _i64p(out)), "trust")
    return int(out[0])


def trustworthiness(original, deformed, n_neighbors: int = 10) -> float:
    """metrics.trustworthiness (metrics.py:74-113)."""
    n = len(original)
    if len(deformed) != n:
        raise ValueError("arrays must have the same length")
    if n <= n_neighbors:
        raise ValueError(f"need more than {n_neighbors} samples")
    total = float(trust_penalty(original, deformed, n_neighbors))
    if total == 0.0:
        return 1.0
    return 1.0 - total / (n * n_neighbors * (2 * n - 3 * n_neighbors - 1) / 2.0)


def subsample(n: int, cap: int = _SUBSAMPLE_CAP):
    """The fixed-seed pick of metrics.py:132-134 / 162-165 (None if n <= cap)."""
    if n <= cap:
        return None
    return np.random.Generator(np.random.PCG64(_SUBSAMPLE_SEED)).choice(n, size=cap, replace=False)


def orthogonal_ordering(original, deformed, sample_cap: int = _SUBSAMPLE_CAP) -> float:
    """metrics.orthogonal_ordering (metrics.py:116-144)."""
    o, m = _f64(original).reshape(-1, 2), _f64(deformed).reshape(-1, 2)
    n = len(o)
    if len(m) != n:
        raise ValueError("arrays must have the same length")
    if n < 2:
        return 1.0
    pick = subsample(n, sample_cap)
    if pick is not None:
        o, m, n = np.ascontiguousarray(o[pick]), np.ascontiguousarray(m[pick]), sample_cap
    out = np.zeros(1, dtype=np.int64)
    _check(_metric_lib().orc_order_pairs(_p(o), _p(m), n, _i64p(out)), "order")
    return int(out[0]) / (n * (n - 1) / 2)


def record_for_frame(original, positions, k: int, full: bool = False, n_neighbors: int = 10):
    """metrics.record_for_frame (metrics.py:147-168) -> (binned_stddev, overplotting,
    trustworthiness | None, ordering | None)."""
    trust = order = None
    o, m = _f64(original).reshape(-1, 2), _f64(positions).reshape(-1, 2)
    if full and len(m) > n_neighbors:
        pick = subsample(len(o))
        if pick is not None:
            o, m = np.ascontiguousarray(o[pick]), np.ascontiguousarray(m[pick])
        trust = trustworthiness(o, m, n_neighbors)
        order = orthogonal_ordering(o, m)
    pos = _f64(positions).reshape(-1, 2)
    return (binned_stddev(pos, k), overplotting(pos, k) if len(pos) else 0.0, trust, order)


# --------------------------------------------------------------- deform_background
def background_splat(targets, values, k: int):
    """encodings.py:141-156 -> (out, covered): the weight-normalised bilinear splat
    before the nearest-covered fill."""
    t = _f64(targets).reshape(-1, 2)
    v = _f64(values).ravel()
    s = 1 << k
    out = np.empty((s, s))
    cov = np.empty((s, s), dtype=np.uint8)
    L = lib()
    L.orc_background_splat.argtypes = [_dp, _dp, ctypes.c_int, _dp, ctypes.POINTER(ctypes.c_ubyte)]
    _check(L.orc_background_splat(_p(t), _p(v), k, _p(out), cov.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte))),
           "background_splat")
    return out, cov.astype(bool)


def background_fill(out, covered):
    """encodings.py:157-159: uncovered pixels copy their nearest covered pixel, through
    the reference's own dependency (scipy.ndimage.distance_transform_edt)."""
    from scipy.ndimage import distance_transform_edt

    out = out.copy()
    if not covered.all():
        dist, (jn, in_) = distance_transform_edt(~covered, return_indices=True)
        out[~covered] = out[jn[~covered], in_[~covered]]
    else:
        dist = np.zeros(covered.shape)
    return out, dist


def deform_background(targets, values, k: int):
    """encodings.deform_background (encodings.py:124-162) from the mapped source pixel
    coordinates and the iteration-0 density values -> (values, distance of every pixel
    to its nearest covered pixel)."""
    out, cov = background_splat(targets, values, k)
    return background_fill(out, cov)
