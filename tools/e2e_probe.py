"""Where the C2 end-to-end call spends its time: pageable H2D of the float64 input, the
device run, the float64 D2H of the result (wall clock, medians of 10).
  python tools/e2e_probe.py"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_06513_b200 as P  # noqa: E402
from bench import four_cluster  # noqa: E402
from paper_2408_06513_b200 import _device as D  # noqa: E402


def med(f, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


host = four_cluster().astype(np.float64)
params = P.RegularizationParams(k=10, kernel_size=8, iterations=10, frame_cap=2)
ds = P.ScatterDataset(positions=host)
dev = torch.empty(host.size, dtype=torch.float32, device="cuda")
pinned = torch.empty(host.shape, dtype=torch.float64, pin_memory=True)
pinned.numpy()[:] = host
g64 = torch.empty(host.shape, dtype=torch.float64, device="cuda")
for _ in range(3):
    P.run(ds, params, store_fields=False).frame(10)
print("h2d staged (to_device)    %.3f ms" % med(lambda: D.to_device(host, out=dev)))
print("h2d to_device, pinned in  %.3f ms" % med(lambda: D.to_device(pinned.numpy(), out=dev)))
g64b = torch.empty(host.shape, dtype=torch.float64, device="cuda")
print("h2d pageable f64          %.3f ms" % med(lambda: g64b.copy_(torch.from_numpy(host), non_blocking=True)))
out64 = np.empty_like(host)
from paper_2408_06513_b200 import _lib
lib = _lib.load()
print("d2h staged widen          %.3f ms" % med(lambda: lib.inim_d2h_widen(D.ptr(dev), out64.ctypes.data, dev.numel(), D.stream())))
print("h2d pinned f64            %.3f ms" % med(lambda: g64.copy_(pinned, non_blocking=True)))
print("d2h f32->f64 pinned       %.3f ms" % med(lambda: D.to_host64(dev)))
print("host memcpy 16 MB         %.3f ms" % med(lambda: np.copyto(pinned.numpy(), host)))
print("run + frame(10)           %.3f ms" % med(lambda: P.run(ds, params, store_fields=False).frame(10)))
