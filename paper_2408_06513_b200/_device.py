"""Device plumbing: CUDA availability, streams, workspace cache, host<->device moves.

PyTorch only allocates memory and supplies the stream; all arithmetic is in
libinim.so.  Nothing here computes on the CPU: without a CUDA device the package
raises instead of falling back.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_ws_cache: dict = {}


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2408_06513_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return _lib.load()


MAX_K = 15  # include/inim.h INIM_MAX_K: 32768^2 = 2^30 pixels


def check_grid(k: int) -> int:
    """The device path covers grids up to 2^15 x 2^15 (int32 pixel indices; the eight fp32
    tables alone take 32 GiB there).  The reference has no upper bound of its own but
    allocates float64 (s, s) arrays, eight tables = 8 * 4^k * 8 bytes (256 GiB at k = 16):
    past k = 15 it runs out of memory, and so does this path, with the same exception
    type numpy raises."""
    k = int(k)
    if k > MAX_K:
        raise MemoryError(f"a 2^{k} x 2^{k} grid exceeds the device path (k <= {MAX_K}); the reference's "
                          f"float64 tables would need {8 * 8 * 4 ** k / 2 ** 30:.0f} GiB")
    return k


def device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(None)
    return ctypes.c_void_p(t.data_ptr())


def workspace(k: int, n: int = 0) -> torch.Tensor:
    """Grow-only per-device workspace for a 2^k grid and n points."""
    lib = require_cuda()
    check_grid(k)
    need = int(lib.inim_workspace_bytes(int(k), int(n), 1))
    if need == 0:
        raise ValueError(f"k={k} out of range")
    key = torch.cuda.current_device()
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            torch.cuda.synchronize()
            lib.inim_clear_graph_cache()
        ws = torch.empty(need, dtype=torch.uint8, device=device())
        _ws_cache[key] = ws
    return ws


def to_device(a, dtype=torch.float32, out: torch.Tensor = None) -> torch.Tensor:
    """Host array (any float dtype) -> contiguous device tensor of `dtype` (float32:
    optionally cast straight into `out`, a contiguous float32 tensor of a.size)."""
    if isinstance(a, torch.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    if dtype == torch.float32:
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        if out is None:
            out = torch.empty(arr.shape, dtype=torch.float32, device=device())
        elif not (out.dtype == torch.float32 and out.is_contiguous() and out.numel() == arr.size):
            raise ValueError("to_device: `out` must be a contiguous float32 tensor of the same size")
        lib = require_cuda()
        src = torch.from_numpy(arr)
        if arr.size and src.is_pinned():
            # page-locked float64: one DMA, narrowed on the device (no host work)
            dev64 = src.to(device(), non_blocking=True)
            _lib.check(lib.inim_cast_f64_to_f32(ptr(dev64), ptr(out), arr.size, stream()), "cast")
            return out
        # pageable float64: narrowed on the host cores in chunks while the DMA engine
        # moves the previous chunk (inim_h2d_narrow, page-locked slots, half the bytes)
        _lib.check(lib.inim_h2d_narrow(arr.ctypes.data, ptr(out), arr.size, stream()), "h2d")
        return out
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(device())


def to_host64(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> host float64 ndarray (widened on the device)."""
    if t.dtype == torch.float64:
        host = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
        host.copy_(t.detach())
        return host.numpy()
    lib = require_cuda()
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    _lib.check(lib.inim_cast_f32_to_f64(ptr(t), ptr(out), t.numel(), stream()), "cast")
    # page-locked destination from torch's caching host allocator (reused across calls):
    # the copy is one DMA instead of a staged pageable copy into fresh pages
    host = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(out)
    return host.numpy()


def to_host64_async(t: torch.Tensor):
    """Start the device->host float64 copy of a float32 device tensor; returns
    (pinned host tensor, CUDA event).  The host data is valid once the event completes."""
    lib = require_cuda()
    t = t.contiguous()
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    _lib.check(lib.inim_cast_f32_to_f64(ptr(t), ptr(out), t.numel(), stream()), "cast")
    host = torch.empty(t.shape, dtype=torch.float64, pin_memory=True)
    host.copy_(out, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return host, ev
