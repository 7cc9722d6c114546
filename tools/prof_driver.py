"""Small fixed workloads for ncu captures (run under gpurun).

  python tools/prof_driver.py iter       # 2 eager iterations of the 1M / 1024^2 workload
  python tools/prof_driver.py integral   # inim_integral_set at 4096^2 (and 16384^2 with --big)
  python tools/prof_driver.py splom      # a batched SPLOM run (PROF_PLOTS plots, PROF_ITERS iterations)
"""

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import four_cluster  # noqa: E402
from paper_2408_06513_b200 import _device as D  # noqa: E402
from paper_2408_06513_b200 import _lib  # noqa: E402


ITER = int(os.environ.get("PROF_ITERS", "2"))


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "iter"
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    if mode in ("iter", "iter3"):
        if mode == "iter3":  # 16M points / 4096^2
            from bench import c3_points
            host, k = c3_points(16_000_000), 12
        else:
            host, k = four_cluster(), 10
        n = len(host)
        pts = torch.from_numpy(host.astype(np.float32)).to(dev)
        ws = torch.empty(int(lib.inim_workspace_bytes(k, n, 1)), dtype=torch.uint8, device=dev)
        for _ in range(2):
            _lib.check(lib.inim_run_uncached(D.ptr(pts), n, k, 8, 0.0, ITER, 0.0, None, None, None, None, None,
                                             D.ptr(ws), D.stream()), "run")
    elif mode == "splom":  # one batched run of PROF_PLOTS C4 plots (500k points, 1024^2)
        from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot

        nplots = int(os.environ.get("PROF_PLOTS", "32"))
        cfg = SplomConfig(nplots=nplots, points=500_000, k=10, kernel_size=8, iterations=ITER)
        job = DeviceSplom(cfg, range(nplots))
        job.load(lambda i: splom_plot(i % 8, cfg.points))
        for _ in range(2):
            job.run()
    else:
        ks = [12] + ([14] if "--big" in sys.argv else [])
        for k in ks:
            s = 1 << k
            d = torch.rand((s, s), device=dev) * 10
            t8 = torch.empty((8, s, s), device=dev)
            tot = torch.empty(1, dtype=torch.float64, device=dev)
            ws = torch.empty(int(lib.inim_workspace_bytes(k, 0, 1)), dtype=torch.uint8, device=dev)
            for _ in range(2):
                _lib.check(lib.inim_integral_set(D.ptr(d), k, D.ptr(t8), D.ptr(tot), D.ptr(ws), D.stream()), "int")
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
