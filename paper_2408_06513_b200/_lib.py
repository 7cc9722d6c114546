"""ctypes binding of libinim.so (the C ABI declared in include/inim.h).

The shared library is built in-tree (``csrc/Makefile`` -> ``paper_2408_06513_b200/
libinim.so``) for sm_100a.  There is no fallback: if the library or a CUDA device is
missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import re
import subprocess
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libinim.so"
CSRC = PKG_DIR / "csrc"
HEADER = PKG_DIR.parent / "include" / "inim.h"

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_float = ctypes.c_float
c_double = ctypes.c_double
c_size_t = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/inim.h
_SIGS = {
    "inim_version": (ctypes.c_char_p, []),
    "inim_workspace_bytes": (c_size_t, [c_int, c_i64, c_int]),
    "inim_run_batched": (c_int, [c_void_p, c_i64, c_int, c_int, c_int, c_float, c_int, c_float, c_void_p, c_void_p,
                                 c_void_p, c_void_p]),
    "inim_splat": (c_int, [c_void_p, c_int, c_i64, c_int, c_void_p, c_void_p]),
    "inim_smooth_counts": (c_int, [c_void_p, c_int, c_int, c_float, c_void_p, c_void_p, c_void_p]),
    "inim_smooth_grid": (c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "inim_integral_set": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "inim_column_integrals": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "inim_line_scan": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p]),
    "inim_field_from_density": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_void_p]),
    "inim_field_from_tables": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "inim_flat_response": (c_int, [c_int, c_void_p, c_void_p]),
    "inim_flat_response_f64": (c_int, [c_int, c_void_p, c_void_p]),
    "inim_sample": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_i64, c_int, c_void_p, c_void_p]),
    "inim_sample_f64": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_i64, c_int, c_void_p]),
    "inim_sample_t64": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_i64, c_int, c_void_p]),
    "inim_map_points": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int, c_void_p,
                                c_void_p]),
    "inim_tilted_wedges": (c_int, [c_void_p] * 6 + [c_int, c_void_p, c_void_p, c_void_p]),
    "inim_cast_f64_to_f32": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "inim_cast_f32_to_f64": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "inim_h2d_narrow": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "inim_d2h_widen": (c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "inim_iterate": (c_int, [c_void_p, c_void_p, c_i64, c_int, c_int, c_float, c_void_p, c_void_p, c_void_p,
                             c_void_p, c_void_p, c_void_p, c_float, c_void_p, c_void_p, c_void_p]),
    "inim_run": (c_int, [c_void_p, c_i64, c_int, c_int, c_float, c_int, c_float, c_void_p, c_void_p, c_void_p,
                         c_void_p, c_void_p, c_void_p, c_void_p]),
    "inim_run_uncached": (c_int, [c_void_p, c_i64, c_int, c_int, c_float, c_int, c_float, c_void_p, c_void_p,
                                  c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "inim_clear_graph_cache": (None, []),
    "inim_profile_run":(c_int, [c_void_p, c_i64, c_int, c_int, c_float, c_int, c_void_p, c_void_p, c_void_p, c_int,
                                 ctypes.c_char_p, c_int]),
    "inim_run_host": (c_int, [c_void_p, c_void_p, c_i64, c_int, c_int, c_double, c_int]),
    "inim_kernels_per_iteration": (c_int, [c_int]),
    "inim_run_metrics": (c_int, [c_void_p, c_i64, c_int, c_int, c_float, c_int, c_float, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_i64, c_int,
                                 c_void_p, c_void_p]),
    "inim_frame_stats": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "inim_gather_points": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "inim_trust_penalty": (c_int, [c_void_p, c_void_p, c_i64, c_int, c_void_p, c_void_p]),
    "inim_order_pairs": (c_int, [c_void_p, c_void_p, c_i64, c_void_p, c_void_p]),
    "inim_deform_background_scratch_bytes": (c_size_t, [c_int]),
    "inim_deform_background": (c_int, [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "inim_blend_frames": (c_int, [c_void_p, c_int, c_void_p, c_int, c_i64, c_double, c_int, c_void_p, c_void_p]),
}

INIM_EINVAL, INIM_ENOTPOW2, INIM_EKERNEL, INIM_EDRIVER = -1, -2, -3, -4

_lib = None


def declared_symbols() -> list[str]:
    """Every function name declared in include/inim.h."""
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(inim_[a-z0-9_]+)\s*\(", text)))


def build(force: bool = False) -> Path:
    """Compile libinim.so for sm_100a with the in-tree Makefile."""
    srcs = list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cuh")) + [HEADER]
    newest = max(p.stat().st_mtime for p in srcs)
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < newest:
        jobs = str(min(8, os.cpu_count() or 1))
        subprocess.run(["make", "-s", "-j", jobs, "-C", str(CSRC)], check=True)
    return LIB_PATH


def load(path: Path | None = None):
    """Load (once) and type the C ABI.  Raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    # INIM_LIB_PATH: an alternative build of the same ABI (A/B timing experiments)
    p = Path(path) if path else Path(os.environ.get("INIM_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise RuntimeError(f"libinim.so not built ({p}); run paper_2408_06513_b200._lib.build() "
                           "or `make -C paper_2408_06513_b200/csrc` -- there is no CPU fallback")
    lib = ctypes.CDLL(str(p))
    alt = p.resolve() != LIB_PATH.resolve()
    for name, (res, args) in _SIGS.items():
        if alt and not hasattr(lib, name):  # an older build under A/B timing: bind what it has
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class InimError(RuntimeError):
    """A libinim call returned a CUDA error or an argument error."""


def check(rc: int, what: str):
    if rc == 0:
        return
    if rc == INIM_EINVAL:
        raise ValueError(f"{what}: invalid argument")
    if rc == INIM_ENOTPOW2:
        raise ValueError("texture must be square with a power-of-two side")
    if rc == INIM_EKERNEL:
        raise ValueError("kernel_size must be >= 1")
    if rc == INIM_EDRIVER:
        raise InimError(f"{what}: could not resolve cuTensorMapEncodeTiled")
    raise InimError(f"{what}: CUDA error {rc}")
