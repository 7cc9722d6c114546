"""Rasterized sample density on the GPU (drop-in for uncrowd density.py:14-78).

accumulate      -> inim_splat (integer atomics; bit-exact counts)
gaussian_smooth -> inim_smooth_grid (two-pass 6*ks+1-tap FIR, reflect borders)
build_density   -> inim_splat + inim_smooth_counts (+ background)
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import ZeroBackground
from .model import DensityTexture, RegularizationParams, ScatterDataset


def _check_square_pow2(shape, what="grid"):
    if len(shape) != 2 or shape[0] != shape[1] or shape[0] < 1 or shape[0] & (shape[0] - 1):
        raise ValueError(f"{what} must be square with a power-of-two side on the device path")
    return int(shape[0]).bit_length() - 1


def _splat_device(positions: np.ndarray, k: int) -> torch.Tensor:
    """Counts (s, s) int32 on the device; float64 coordinates binned in float64."""
    lib = D.require_cuda()
    s = 1 << D.check_grid(k)
    counts = torch.zeros((s, s), dtype=torch.int32, device=D.device())
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 2)
    if len(pos):
        if (pos < 0).any() or not np.isfinite(pos).all():
            # np.bincount rejects negative (and NaN-derived) bin indices (density.py:25)
            raise ValueError("positions must be finite and non-negative")
        dev = torch.from_numpy(pos).to(D.device())
        _lib.check(lib.inim_splat(D.ptr(dev), 1, len(pos), k, D.ptr(counts), D.stream()), "splat")
    return counts


def accumulate(positions, k: int) -> np.ndarray:
    """Per-pixel sample counts as float64 (density.py:14-27)."""
    counts = _splat_device(np.asarray(positions, dtype=np.float64), k)
    return counts.to(torch.float64).cpu().numpy()


def smoothing_kernel(kernel_size: int) -> np.ndarray:
    """Normalized Gaussian taps, sigma = ks/2, 3*ks taps per side (density.py:30-37).
    (The device kernels build the same taps internally in float64 -> float32.)"""
    radius = 3 * kernel_size
    t = np.arange(-radius, radius + 1, dtype=np.float64) / (kernel_size / 2.0)
    w = np.exp(-0.5 * t * t)
    return w / w.sum()


def gaussian_smooth(grid, kernel_size: int) -> np.ndarray:
    """Horizontal then vertical 6*ks+1-tap pass with reflected borders (density.py:40-51)."""
    if kernel_size < 1:
        raise ValueError("kernel_size must be >= 1")
    g = np.asarray(grid, dtype=np.float64)
    k = _check_square_pow2(g.shape)
    lib = D.require_cuda()
    src = D.to_device(g)
    out = torch.empty_like(src)
    ws = D.workspace(k)
    _lib.check(lib.inim_smooth_grid(D.ptr(src), k, kernel_size, D.ptr(out), D.ptr(ws), D.stream()),
               "gaussian_smooth")
    return D.to_host64(out)


def resolve_background(params: RegularizationParams, n: int) -> float:
    """Explicit background (> 0) or n / 4^k, 1.0 for an empty dataset (density.py:61-70)."""
    if params.background is not None:
        if params.background <= 0:
            raise ZeroBackground("background density must be > 0")
        return float(params.background)
    bg = n / float(1 << (2 * params.k))
    return 1.0 if bg == 0.0 else bg


def build_density(dataset_or_positions, params: RegularizationParams, n: Optional[int] = None) -> DensityTexture:
    """Smoothed counts plus background at every pixel (density.py:54-78)."""
    positions = (dataset_or_positions.positions if isinstance(dataset_or_positions, ScatterDataset)
                 else np.asarray(dataset_or_positions))
    if n is None:
        n = len(positions)
    background = resolve_background(params, n)
    if params.kernel_size < 1:
        raise ValueError("kernel_size must be >= 1")
    lib = D.require_cuda()
    k = params.k
    counts = _splat_device(positions, k)
    d = torch.empty(counts.shape, dtype=torch.float32, device=D.device())
    ws = D.workspace(k)
    _lib.check(lib.inim_smooth_counts(D.ptr(counts), k, params.kernel_size, background, D.ptr(d), D.ptr(ws),
                                      D.stream()), "build_density")
    return DensityTexture(k=k, kernel_size=params.kernel_size, background=background, n=n, device_values=d)
