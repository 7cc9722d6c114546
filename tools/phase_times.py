"""Per-phase durations of the persistent iteration kernel (globaltimer stamps of the
first iteration), for the 1M-point / 1024^2 workload.  Run under gpurun."""

import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import four_cluster  # noqa: E402
from paper_2408_06513_b200 import _device as D  # noqa: E402
from paper_2408_06513_b200 import _lib  # noqa: E402

NAMES = ["splat", "smooth_h", "smooth_v+reduce+lines", "chains", "field", "move"]


def main():
    k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
    lib = _lib.load()
    host = four_cluster(n)
    pts0 = torch.from_numpy(host.astype(np.float32)).cuda()
    pts = pts0.clone()
    ws = torch.empty(int(lib.inim_workspace_bytes(k, n)), dtype=torch.uint8, device="cuda")
    st = torch.zeros(16, dtype=torch.int64, device="cuda")
    acc = np.zeros(len(NAMES))
    reps = 20
    for q in range(reps + 3):
        pts.copy_(pts0)
        rc = lib.inim_run_stamped(D.ptr(pts), n, k, 8, 0.0, 2, D.ptr(ws), D.stream(), D.ptr(st))
        if rc != 1:
            print("persistent path not used:", rc)
            return
        torch.cuda.synchronize()
        t = st.cpu().numpy()[: len(NAMES) + 1].astype(np.float64)
        if q >= 3:
            acc += np.diff(t)
    acc /= reps
    for nm, v in zip(NAMES, acc):
        print(f"{nm:18s} {v / 1e3:8.2f} us")
    print(f"{'total':18s} {acc.sum() / 1e3:8.2f} us")


if __name__ == "__main__":
    main()
