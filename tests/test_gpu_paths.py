"""GPU parity of the specialised kernel paths, one test per instantiation family:

  counts smoothing  the horizontal FIR on packed FFMA2 (broadcast input, shifted tap
                    pairs) is a separate template per kernel_size 1..16 and per tile
                    geometry (compile-time 32 x 128 tiles from 128^2 up, runtime tiles
                    below): every one against the oracle's gaussian_smooth + background
                    (density.py:30-78)
  batch move        the pipelined batch move (cp.async.bulk chunks of 512 point pairs,
                    eight chunks per CTA) at plot sizes that leave partial chunks, a
                    single chunk, a single pair, and CTAs with fewer than eight chunks:
                    against each plot regularized alone and against the oracle
  runtime switches  every INIM_* switch of INTEGRATION.md section 5 leaves single-plot and
                    batched results bit-identical
"""

import numpy as np
import pytest

from conftest import clusters

pytestmark = pytest.mark.gpu

POS_TOL = 2e-5


def maxerr(a, b):
    return float(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)).max())


@pytest.mark.parametrize("ks", list(range(1, 17)))
def test_counts_smoothing_every_kernel_size(P, oracle, ks):
    for k in (8, 6):  # 256^2: compile-time 32 x 128 tiles; 64^2: runtime tile geometry
        pts = clusters(40_000, 100 + ks + k)
        tex = P.build_density(pts, P.RegularizationParams(k=k, kernel_size=ks))
        want, bg = oracle.build_density(pts, k, ks)
        assert tex.background == bg
        assert maxerr(tex.values, want) <= 2e-6 * want.max(), (k, ks)


@pytest.mark.parametrize("points", [2, 34, 1026, 9_000, 70_002])
def test_batch_move_partial_chunks(P, oracle, points):
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot

    iters = 3
    cfg = SplomConfig(nplots=3, points=points, k=8, kernel_size=8, iterations=iters)
    job = DeviceSplom(cfg, range(cfg.nplots))
    job.load(lambda i: splom_plot(i, cfg.points))
    res = job.run().cpu().numpy().astype(np.float64)
    for i in range(cfg.nplots):
        pts = splom_plot(i, cfg.points)
        r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=8, kernel_size=8, iterations=iters),
                  store_fields=False)
        assert maxerr(res[i], r.frame(iters)) <= POS_TOL, (points, i)
        assert maxerr(res[i], oracle.run_positions(pts, 8, 8, iters)[-1]) <= POS_TOL, (points, i)


SWITCH_SCRIPT = """
import sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2408_06513_b200 as P
from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot
host = np.load({inp!r})
r = P.run(P.ScatterDataset(positions=host), P.RegularizationParams(k=10, kernel_size=8, iterations=4),
          store_fields=False)
cfg = SplomConfig(nplots=6, points=70_000, k=9, kernel_size=8, iterations=4, collect_metrics=True)
job = DeviceSplom(cfg, range(cfg.nplots))
job.load(lambda i: splom_plot(i, cfg.points))
pos = job.run().cpu().numpy()
np.savez({out!r}, single=r.frame(4), batch=pos, met=np.asarray(job.metrics(), dtype=np.float64))
"""


@pytest.mark.parametrize("switch", ["INIM_V_EMIT=0", "INIM_MOVE_BULK=0", "INIM_CLEAR_IN_V=0", "INIM_ZREV=0",
                                    "INIM_SORT=0", "INIM_PDL=0"])
def test_runtime_switches_bit_identical(tmp_path, switch):
    """none of the runtime switches changes a result.  One
    single-plot run (sorted path) and one batched SPLOM run with frame statistics, with
    the switch and without, compared bit for bit."""
    import os
    import subprocess
    import sys

    from conftest import ROOT

    np.save(tmp_path / "in.npy", clusters(200_000, 10).astype(np.float64))
    outs = []
    for tag, env in (("base", {}), ("sw", dict([switch.split("=")]))):
        dst = tmp_path / f"{tag}.npz"
        f = tmp_path / f"{tag}.py"
        f.write_text(SWITCH_SCRIPT.format(root=str(ROOT), inp=str(tmp_path / "in.npy"), out=str(dst)))
        run = subprocess.run([sys.executable, str(f)], capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, **env))
        assert run.returncode == 0, run.stderr[-2000:]
        outs.append(np.load(dst))
    for key in ("single", "batch", "met"):
        assert np.array_equal(outs[0][key], outs[1][key]), (switch, key)
