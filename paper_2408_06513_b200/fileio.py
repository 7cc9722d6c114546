"""Binary dumps of device-resident results (drop-in for uncrowd fileio.py:15-125).

The field dump (``INIMFLD\\0``, fileio.py:63-85) is a 16-byte header (magic, u32 k,
u32 iteration, little-endian) followed by the (s, s, 2) float32 targets, row-major, x
before y -- exactly the device field layout, so a field produced on the GPU is written
with one device->host copy of its buffer and read back with one host->device copy,
bit-identical both ways.  ``INIMGRD\\0`` does the same for one scalar table.  The
service's binary positions payload (service.py:170-172) is the f64 frame blend of
transition_positions rounded to float32, computed on the device (inim_blend_frames).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import FormatError, OutOfRangeLevel
from .metrics import MetricRecord
from .model import DeformationField, RegularizationRun

FIELD_MAGIC = b"INIMFLD\x00"
GRID_MAGIC = b"INIMGRD\x00"
_HEADER = struct.Struct("<II")  # k, index (after the 8-byte magic)


def _f32_bytes(t: torch.Tensor) -> bytes:
    """Little-endian float32 bytes of a device float32 tensor (one D2H copy)."""
    host = torch.empty(t.shape, dtype=torch.float32, pin_memory=True)
    host.copy_(t.detach().contiguous())
    return host.numpy().astype("<f4", copy=False).tobytes()


def _field_payload(field: DeformationField) -> bytes:
    if field.device_targets64() is None:  # float32 device field: its own bytes
        return _f32_bytes(field.device_targets())
    return field.targets.astype("<f4").tobytes()  # caller-built float64 targets


def export_field(field: DeformationField, path, iteration: int = 0):
    """Binary field dump: magic, u32 k, u32 iteration, 2 * 4^k float32 (fileio.py:63-70)."""
    payload = _field_payload(field)
    with open(path, "wb") as handle:
        handle.write(FIELD_MAGIC)
        handle.write(_HEADER.pack(field.k, iteration))
        handle.write(payload)


def read_field(path):
    """Inverse of export_field -> (DeformationField, iteration) (fileio.py:73-85).  The
    float32 payload goes to the device as the field's own buffer (exact)."""
    blob = Path(path).read_bytes()
    if blob[:8] != FIELD_MAGIC:
        raise FormatError(f"bad magic in {path}")
    if len(blob) < 16:
        raise FormatError(f"truncated header in {path}")
    k, iteration = _HEADER.unpack_from(blob, 8)
    size = 1 << k
    expected = 16 + 2 * size * size * 4
    if len(blob) != expected:
        raise FormatError(f"expected {expected} bytes for k={k}, got {len(blob)}")
    host = np.frombuffer(blob, dtype="<f4", offset=16).reshape(size, size, 2)
    if torch.cuda.is_available():
        dev = torch.from_numpy(host.astype(np.float32)).to(D.device())
        return DeformationField(k=k, device_targets=dev), iteration
    # no device: the caller still gets the reference's float64 view of the payload
    return DeformationField(targets=host.astype(np.float64), k=k), iteration


def export_grid(values, path, k: int, index: int = 0):
    """Debug dump of one scalar table in the field-dump layout (fileio.py:88-93).
    Device float32 tensors are written with one D2H copy."""
    if isinstance(values, torch.Tensor) and values.dtype == torch.float32:
        payload = _f32_bytes(values)
    else:
        payload = np.asarray(values).astype("<f4").tobytes()
    with open(path, "wb") as handle:
        handle.write(GRID_MAGIC)
        handle.write(_HEADER.pack(k, index))
        handle.write(payload)


def read_grid(path):
    """Inverse of export_grid -> (values (s, s) float64, index) (fileio.py:96-104)."""
    blob = Path(path).read_bytes()
    if blob[:8] != GRID_MAGIC:
        raise FormatError(f"bad magic in {path}")
    if len(blob) < 16:
        raise FormatError(f"truncated header in {path}")
    k, index = _HEADER.unpack_from(blob, 8)
    size = 1 << k
    if len(blob) != 16 + size * size * 4:
        raise FormatError("payload size does not match header")
    values = np.frombuffer(blob, dtype="<f4", offset=16).astype(np.float64)
    return values.reshape(size, size), index


def write_metrics(records, path):
    """Line-delimited metric records, stable key order (fileio.py:107-111)."""
    with open(path, "w", encoding="utf-8") as handle:
        for record in records:
            handle.write(record.to_json_line() + "\n")


def read_metrics(path) -> list:
    with open(path, "r", encoding="utf-8") as handle:
        return [MetricRecord.from_json_line(line) for line in handle if line.strip()]


def _frame_device(run: RegularizationRun, t: int):
    """(tensor, is_f64): frame 0 is the caller's float64 layout, later frames the run's
    float32 device frames (recomputed on the device when thinned away)."""
    if t == 0:
        return torch.from_numpy(np.ascontiguousarray(run.original.positions, dtype=np.float64)).to(D.device()), 1
    if t not in run._dev_frames:
        run.frame(t)  # recompute (device) and cache
        if t not in run._dev_frames:
            return torch.from_numpy(run.frame(t)).to(D.device()), 1
    return run._dev_frames[t].contiguous(), 0


def positions_payload(run: RegularizationRun, level: float) -> bytes:
    """The service's binary positions response (service.py:166-172):
    transition_positions(run, level).astype('<f4').tobytes(), blended on the device in
    float64 in the reference's operation order (regularize.py:83-93)."""
    lib = D.require_cuda()
    top = run.iterations
    if not 0.0 <= level <= top:
        raise OutOfRangeLevel(f"level {level} outside [0, {top}]")
    low, high = int(np.floor(level)), int(np.ceil(level))
    n = run.original.n
    if n == 0:
        return b""
    lo, lo64 = _frame_device(run, low)
    hi, hi64 = _frame_device(run, high)
    frac = 0.0 if low == high else level - low
    out = torch.empty((n, 2), dtype=torch.float32, device=D.device())
    _lib.check(lib.inim_blend_frames(D.ptr(lo), lo64, D.ptr(hi), hi64, 2 * n, float(frac), int(low == high),
                                     D.ptr(out), D.stream()), "positions_payload")
    return _f32_bytes(out)
