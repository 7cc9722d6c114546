"""SPLOM step through DeviceSplom.run_host (page-locked float32 host buffers, chunked
copies overlapping the batched runs) for several chunk / lead sizes, median wall time:
  python tools/splom_e2e_probe.py [plots]"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot  # noqa: E402

plots = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = SplomConfig(nplots=plots, points=500_000, k=10, kernel_size=8, iterations=10, max_batch=256)
job = DeviceSplom(cfg, range(plots))
cache = {}
job.load(lambda i: cache.setdefault(i % 16, splom_plot(i % 16, cfg.points)))
host_in = torch.empty(tuple(job.inputs.shape), dtype=torch.float32).pin_memory()
host_in.copy_(job.inputs.cpu())
host_out = torch.empty_like(host_in).pin_memory()
for chunk, lead in [(96, 8), (96, 0), (64, 32), (96, 4)]:
    def call():
        job.run_host(host_in, host_out, chunk=chunk, lead=lead)
        torch.cuda.current_stream().synchronize()
    for _ in range(2):
        call()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    dt = statistics.median(ts)
    print(f"chunk={chunk} lead={lead} ms={dt * 1e3:.2f} plot-iters/s={plots * 10 / dt:.0f}")
