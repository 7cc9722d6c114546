"""Visual encodings of the deformation on the GPU (drop-in for uncrowd encodings.py).

deform_grid / deform_contours push every polyline vertex through the same composed
per-iteration fields the samples go through (map_through, regularize.py:96-109), all
vertices of all polylines in ONE batch per field, so a vertex coincident with a sample
lands exactly on that sample's deformed position (the run's float32 move arithmetic).

deform_background (encodings.py:124-162) maps every source pixel through the fields,
then inim_deform_background splats the iteration-0 density with bilinear weights as a
deterministic gather in the reference's np.add.at order, normalises, and fills the
uncovered pixels from their nearest covered pixel (exact Euclidean distance transform).

Contour extraction itself (extract_contours: skimage marching squares) is host
geometry outside the hot path; deform_contours accepts the
reference's ContourSet as well as this module's.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _device as D
from . import _lib
from .model import DensityTexture, RegularizationRun, unit_coordinates
from .regularize import map_through, map_through_device

DEFAULT_SPACING = 32  # pixels between grid lines at k = 10
DEFAULT_SUBDIVISION = 8  # sampled points per grid cell edge
DEFAULT_LEVEL_FRACTIONS = (1.0 / 16.0, 1.0 / 4.0, 1.0 / 2.0)


@dataclass(frozen=True)
class GridOverlay:
    polylines: list  # list of (m, 2) float arrays in [0,1]^2
    spacing: int
    subdivision: int


@dataclass(frozen=True)
class ContourSet:
    polylines: list  # list of (m, 2) float arrays
    line_levels: list  # density level of each polyline
    levels: list  # the requested level set


@dataclass(frozen=True)
class BackgroundTexture:
    values: np.ndarray  # (2**k, 2**k) resampled original density
    k: int
    value_range: tuple  # (min, max) of the source density
    transfer: str = "luminance"  # named preset, not part of correctness


def _fields_of(run_or_field):
    if isinstance(run_or_field, RegularizationRun):
        return run_or_field.fields
    return [run_or_field]


def _map_batch(fields, lines, upto):
    """map_through of several polylines as one concatenated batch, split back."""
    if not lines:
        return []
    sizes = [len(line) for line in lines]
    allpts = np.concatenate([np.asarray(line, dtype=np.float64).reshape(-1, 2) for line in lines])
    mapped = map_through(fields, allpts, upto)
    return np.split(mapped, np.cumsum(sizes)[:-1])


def deform_grid(run_or_field, spacing: int = DEFAULT_SPACING, subdivision: int = DEFAULT_SUBDIVISION,
                upto: Optional[int] = None) -> GridOverlay:
    """Regular grid polylines mapped through the deformation (encodings.py:55-83)."""
    if spacing < 2:
        raise ValueError("spacing must be >= 2 pixels")
    if subdivision < 1:
        raise ValueError("subdivision must be >= 1")
    fields = _fields_of(run_or_field)
    k = fields[0].k if fields else 10
    size = 1 << k
    pixel_marks = np.arange(0, size + 1, spacing)  # domain edges included
    line_positions = pixel_marks / size
    cells = len(pixel_marks) - 1
    ticks = np.linspace(0.0, line_positions[-1], cells * subdivision + 1)
    lines = []
    for pos in line_positions:
        lines.append(np.column_stack([ticks, np.full_like(ticks, pos)]))  # horizontal
        lines.append(np.column_stack([np.full_like(ticks, pos), ticks]))  # vertical
    return GridOverlay(polylines=_map_batch(fields, lines, upto), spacing=spacing, subdivision=subdivision)


def default_levels(density: DensityTexture) -> list:
    """Levels at fixed fractions of the density excess over the background
    (encodings.py:86-90)."""
    peak = float(density.values.max())
    base = density.background
    return [base + f * (peak - base) for f in DEFAULT_LEVEL_FRACTIONS]


def extract_contours(density: DensityTexture, levels: Sequence[float]) -> ContourSet:
    """Marching-squares isolines (encodings.py:93-112) are skimage host geometry, not
    part of this device build; build the ContourSet with the
    reference and pass it to deform_contours."""
    raise NotImplementedError("extract_contours (skimage marching squares) is not part of the device build; "
                              "use the reference's extract_contours and this module's deform_contours")


def deform_contours(contours, run_or_field, upto: Optional[int] = None) -> ContourSet:
    """Map every contour vertex through the composed fields; levels stay
    (encodings.py:115-121)."""
    fields = _fields_of(run_or_field)
    mapped = _map_batch(fields, list(contours.polylines), upto)
    return ContourSet(polylines=mapped, line_levels=list(contours.line_levels), levels=list(contours.levels))


def background_sources(run: RegularizationRun, upto: Optional[int] = None) -> torch.Tensor:
    """Every source pixel coordinate (unit_coordinates, row-major) pushed through the
    run's fields: float32 device (m, 2) (encodings.py:137-139)."""
    fields = run.fields if upto is None else run.fields[:upto]
    k = run.params.k
    X, Y = unit_coordinates(k)
    src = torch.from_numpy(np.column_stack([X.ravel(), Y.ravel()]).astype(np.float32)).to(D.device())
    if any(f.device_targets64() is not None for f in fields):  # caller-built float64 fields
        return torch.from_numpy(map_through(fields, src.double().cpu().numpy()).astype(np.float32)).to(D.device())
    return map_through_device(fields, src)


def deform_background(run: RegularizationRun, upto: Optional[int] = None) -> BackgroundTexture:
    """Original (iteration-0) density carried to the deformed domain
    (encodings.py:124-162): bilinear splat of every source pixel's value at its mapped
    position, weight-normalised, uncovered pixels from their nearest covered pixel."""
    lib = D.require_cuda()
    from .density import build_density

    density = build_density(run.frame(0), run.params)
    k = density.k
    if k < 1:
        raise ValueError("deform_background needs k >= 1")
    s = 1 << k
    targets = background_sources(run, upto)
    values = density.device_values().to(torch.float32).contiguous()
    out = torch.empty((s, s), dtype=torch.float64, device=D.device())
    vrange = torch.empty(2, dtype=torch.float32, device=D.device())
    nbytes = int(lib.inim_deform_background_scratch_bytes(k))
    if nbytes == 0:
        D.check_grid(k)
        raise ValueError(f"deform_background: k={k} out of range")
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=D.device())
    _lib.check(lib.inim_deform_background(D.ptr(targets), D.ptr(values), k, D.ptr(out), D.ptr(vrange),
                                             D.ptr(scratch), D.stream()), "deform_background")
    vmin, vmax = (float(v) for v in vrange.cpu().tolist())
    return BackgroundTexture(values=D.to_host64(out), k=k, value_range=(vmin, vmax))
