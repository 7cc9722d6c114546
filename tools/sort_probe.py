"""How much does spatial point order buy the move / splat?  Profiles one run of the
C2 and C3 workloads with the input points in generation order and pre-sorted (host)
by a cell key.  python tools/sort_probe.py  (under gpurun)"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import c3_points, four_cluster  # noqa: E402
from paper_2408_06513_b200 import _device as D  # noqa: E402
from paper_2408_06513_b200 import _lib  # noqa: E402


def morton(ix, iy, bits):
    key = np.zeros_like(ix, dtype=np.int64)
    for b in range(bits):
        key |= ((ix >> b) & 1) << (2 * b)
        key |= ((iy >> b) & 1) << (2 * b + 1)
    return key


def profile(lib, host, k, iters=10, reps=3):
    n = len(host)
    pts0 = torch.from_numpy(host.astype(np.float32)).cuda()
    pts = pts0.clone()
    ws = torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device="cuda")
    cap = 64 * iters
    ms = (ctypes.c_float * cap)()
    names = ctypes.create_string_buffer(cap * 24)
    acc = {}
    for r in range(reps + 1):
        pts.copy_(pts0)
        cnt = lib.inim_profile_run(D.ptr(pts), n, k, 8, 0.0, iters, D.ptr(ws), D.stream(), ms, cap, names, len(names))
        if r == 0:
            continue
        for nm, v in zip(names.value.decode().split("\n")[:cnt], ms[:cnt]):
            a = acc.setdefault(nm, [0.0, 0])
            a[0] += v
            a[1] += 1
    return {nm: 1e3 * v[0] / v[1] for nm, v in acc.items()}


def main():
    lib = _lib.load()
    for label, host, k in (("C2", four_cluster(), 10), ("C3", c3_points(16_000_000), 12)):
        s = 1 << k
        ix = np.minimum((host[:, 0] * s).astype(np.int64), s - 1)
        iy = np.minimum((host[:, 1] * s).astype(np.int64), s - 1)
        variants = [("input order", host)]
        for cell in (64, 8, 1):
            key = morton(ix // cell, iy // cell, k)
            variants.append((f"sorted {cell}px cells", host[np.argsort(key, kind="stable")]))
        for name, h in variants:
            prof = profile(lib, np.ascontiguousarray(h), k)
            print(f"{label} {name:22s} " + "  ".join(f"{nm}={v:.1f}" for nm, v in prof.items()), flush=True)


if __name__ == "__main__":
    main()
