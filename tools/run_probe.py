"""Graph-replayed inim_run time vs iteration count (per-run overhead = intercept,
per-iteration cost = slope), 1M four-cluster points on 1024^2, L2 flushed.
  python tools/run_probe.py            (INIM_SORT=0 to compare without the point sort)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import four_cluster, c3_points  # noqa: E402
from paper_2408_06513_b200 import _device as D, _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
big = "c3" in sys.argv
host, k = (c3_points(16_000_000), 12) if big else (four_cluster(), 10)
n = len(host)
pin = torch.from_numpy(host.astype(np.float32)).to(dev)
pts = torch.empty_like(pin)
ws = torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device=dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
st = D.stream()
rows = []
for T in (1, 2, 5, 10, 20):
    def go():
        pts.copy_(pin)
        _lib.check(lib.inim_run(D.ptr(pts), n, k, 8, 0.0, T, 0.0, None, None, None, None, None, D.ptr(ws), st), "run")
    for _ in range(3):
        go()
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        go()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    rows.append((T, float(np.median(ts))))
    print(f"T={T:3d}  {rows[-1][1]:9.1f} us", flush=True)
Ts = np.array([r[0] for r in rows], float)
us = np.array([r[1] for r in rows])
slope, icpt = np.polyfit(Ts, us, 1)
print(f"per iteration {slope:.1f} us, per run {icpt:.1f} us")
