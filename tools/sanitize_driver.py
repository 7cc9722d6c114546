"""Small workloads that launch every libinim kernel once or a few times, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck) on the GPU box:
  compute-sanitizer --tool memcheck python tools/sanitize_driver.py
Sizes are tiny (the tools slow kernels down by 10-100x)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_06513_b200 as P  # noqa: E402


def main():
    rng = np.random.default_rng(3)
    pts = np.clip(rng.normal(0.4, 0.1, size=(20_000, 2)), 0, 1).astype(np.float32).astype(np.float64)
    k = 8
    P.accumulate(pts, k)
    dens = P.build_density(pts, P.RegularizationParams(k=k, kernel_size=4, iterations=1))
    tabs = P.build_integral_set(dens)
    field = P.build_field(tabs)
    P.sample_field(field, pts)
    P.iterate_once(pts, P.RegularizationParams(k=k, kernel_size=4, iterations=1))
    for mode in ("none", "basic", "full"):
        r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=k, kernel_size=8, iterations=3),
                  collect_metrics=mode)
        r.frame(3)
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=k, kernel_size=8, iterations=3,
                                                                      stop="displacement", epsilon=1e-3))
    P.map_through(r, pts[:100])
    P.deform_grid(r)
    P.deform_background(r)
    big = np.clip(rng.normal(0.5, 0.15, size=(70_000, 2)), 0, 1).astype(np.float32).astype(np.float64)
    r = P.run(P.ScatterDataset(positions=big), P.RegularizationParams(k=9, kernel_size=8, iterations=3))  # sorted path
    r.frame(3)
    d = rng.random((4096, 4096)) * 3  # the TMA-ring reduce and the 32 x 128 tile geometry
    P.build_integral_set(d)
    P.build_density(pts, P.RegularizationParams(k=7, kernel_size=20))  # runtime-tap smoothing
    P.gaussian_smooth(rng.random((16, 16)), 12)                         # taps folded onto one period
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot
    cfg = SplomConfig(nplots=3, points=70_000, k=8, kernel_size=8, iterations=3, collect_metrics=True)
    job = DeviceSplom(cfg, range(3))  # the batched run (plot index in grid.z), sorted path
    job.load(lambda i: splom_plot(i, cfg.points))
    job.run()
    job.metrics()
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
