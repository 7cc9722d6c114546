"""Bit-identity of the SPLOM batch under two environment settings of one build (e.g. the
pipelined vs grid-stride batch move):
  python tools/bitcheck_splom.py INIM_MOVE_BULK=0 INIM_MOVE_BULK=4"""
import os
import subprocess
import sys
import textwrap
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
SCRIPT = textwrap.dedent("""
    import sys, numpy as np
    sys.path.insert(0, {root!r})
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot
    cfg = SplomConfig(nplots=12, points=500_001 - 1, k=10, kernel_size=8, iterations=10, collect_metrics=True)
    job = DeviceSplom(cfg, range(12))
    job.load(lambda i: splom_plot(i, cfg.points))
    out = job.run().cpu().numpy()
    np.savez({path!r}, pos=out, met=np.asarray(job.metrics(), dtype=np.float64))
""")


def run(env_kv, path):
    env = dict(os.environ)
    k, v = env_kv.split("=", 1)
    env[k] = v
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), path=path)], env=env, check=True)


if __name__ == "__main__":
    import numpy as np
    a, b = sys.argv[1], sys.argv[2]
    run(a, "/tmp/bs_a.npz")
    run(b, "/tmp/bs_b.npz")
    A, B = np.load("/tmp/bs_a.npz"), np.load("/tmp/bs_b.npz")
    for key in A.files:
        same = np.array_equal(A[key], B[key])
        print(key, "bit-identical" if same else f"DIFFER max {np.abs(A[key] - B[key]).max():.3e}")
