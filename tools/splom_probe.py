"""SPLOM batch step time (C4 plots, 1024^2, 10 iterations) for several batch sizes (plots
per batched launch), L2 flushed, CUDA events:  python tools/splom_probe.py [plots] [max_batch ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot  # noqa: E402

plots = int(sys.argv[1]) if len(sys.argv) > 1 else 256
variants = [int(v) for v in sys.argv[2:]] or [256, 64]
cache = {}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for S in variants:
    cfg = SplomConfig(nplots=plots, points=500_000, k=10, kernel_size=8, iterations=10, max_batch=S)
    job = DeviceSplom(cfg, range(plots))
    job.load(lambda i: cache.setdefault(i % 16, splom_plot(i % 16, cfg.points)))
    for _ in range(3):
        job.run()
    ts = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        job.run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"max_batch={S} plots={plots} ms={np.median(ts):.2f} plot-iters/s={plots * 10 / np.median(ts) * 1e3:.0f}",
          flush=True)
    del job
    torch.cuda.empty_cache()
