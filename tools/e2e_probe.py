"""Where does the end-to-end (public API, host buffers) time go?  python tools/e2e_probe.py [c2|c3]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_06513_b200 as P  # noqa: E402
from bench import c3_points, four_cluster  # noqa: E402
from paper_2408_06513_b200 import _device as D  # noqa: E402


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c2"
    host, k = (four_cluster(), 10) if which == "c2" else (c3_points(16_000_000), 12)
    n = len(host)
    pinned = torch.empty((n, 2), dtype=torch.float64).pin_memory()
    pinned.numpy()[:] = host
    pos = pinned.numpy()
    params = P.RegularizationParams(k=k, kernel_size=8, iterations=10, frame_cap=2)
    for rep in range(4):
        t = [time.perf_counter()]
        ds = P.ScatterDataset(positions=pos)
        t.append(time.perf_counter())
        dev = D.to_device(pos)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        r = P.run(ds, params, store_fields=False)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        out = r.frame(10)
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        print(f"{which} rep{rep}: dataset {d[0]:.2f} ms  to_device {d[1]:.2f} ms  run {d[2]:.2f} ms  "
              f"frame->host {d[3]:.2f} ms  total {sum(d) - d[1]:.2f} ms", flush=True)
        del dev, out


if __name__ == "__main__":
    main()
