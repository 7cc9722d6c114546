"""Layout metrics (metrics.py:46-168): the CPU oracle pinned to golden values recorded
from the unmodified reference, and the host-side integer -> float formulas of the
drop-in (paper_2408_06513_b200.metrics).  CPU only.

Bars: overplotting, trustworthiness, ordering are exact (integer numerators and the
reference's own float formulas); binned_stddev within 1e-12 relative (the oracle and
the device path round the exact variance once, numpy's std accumulates a few ulps).
"""

import json

import numpy as np
import pytest

STD_REL = 1e-12


def test_occupancy_golden(oracle, golden):
    g = golden("metrics")
    for k in (2, 4, 6, 8):
        pts = g[f"occ_pts_k{k}"]
        assert oracle.overplotting(pts, k) == g[f"occ_over_k{k}"]
        assert oracle.binned_stddev(pts, k) == pytest.approx(float(g[f"occ_binned_k{k}"]), rel=STD_REL, abs=0)
    assert oracle.binned_stddev(g["occ_uniform"], 4) == g["occ_binned_uniform"] == 0.0
    assert oracle.overplotting(g["occ_uniform"], 4) == g["occ_over_uniform"] == 0.0


def test_neighbourhood_golden(oracle, golden):
    g = golden("metrics")
    o, m = g["nb_orig"], g["nb_moved"]
    assert oracle.trustworthiness(o, m, 10) == g["nb_trust10"]
    assert oracle.trustworthiness(o, m, 3) == g["nb_trust3"]
    assert oracle.orthogonal_ordering(o, m) == g["nb_order"]
    assert oracle.trustworthiness(o, o, 10) == g["nb_trust_self"] == 1.0
    assert oracle.orthogonal_ordering(o, o) == g["nb_order_self"] == 1.0
    assert oracle.orthogonal_ordering(g["nb_big"], g["nb_bigm"]) == g["nb_order_big"]
    assert oracle.orthogonal_ordering(g["nb_big"], g["nb_bigm"], 1000) == g["nb_order_big_cap"]


def test_run_records_golden(oracle, golden):
    """record_for_frame on the reference's own run frames (10k points: the 4096-row
    fixed-seed subsample) reproduces the reference's run(collect_metrics='full')."""
    g = golden("metrics")
    frames, k = g["run_frames"], int(g["run_k"])
    for t in range(len(frames)):
        b, o, tr, od = oracle.record_for_frame(frames[0], frames[t], k, full=True)
        assert b == pytest.approx(float(g["run_binned"][t]), rel=STD_REL, abs=0)
        assert o == g["run_over"][t]
        assert tr == g["run_trust"][t]
        assert od == g["run_order"][t]


def test_host_formulas_match_numpy(rng):
    """The drop-in's integer -> float conversions against numpy's own std on integer
    bin counts, and the reference's closed forms."""
    from paper_2408_06513_b200 import metrics as M

    for k in (2, 3, 5, 8):
        nb = ((1 << k) // 4) ** 2
        bins = rng.integers(0, 50, size=nb)
        got = M.stddev_from_stats(int((bins.astype(np.int64) ** 2).sum()), int(bins.sum()), k)
        assert got == pytest.approx(float(bins.std()), rel=STD_REL, abs=1e-300)
    assert M.stddev_from_stats(16 * 9, 16 * 3, 4) == 0.0  # every bin holds 3
    assert M.overplotting_from_stats(7, 10) == 0.3
    assert M.trust_from_penalty(0, 100, 10) == 1.0
    n, nn, pen = 600, 10, 12345
    assert M.trust_from_penalty(pen, n, nn) == 1.0 - float(pen) / (n * nn * (2 * n - 3 * nn - 1) / 2.0)
    assert M.ordering_from_pairs(10, 5) == 1.0


def test_subsample_rows_match_reference_generator():
    from paper_2408_06513_b200 import metrics as M

    assert M.subsample_rows(4096) is None
    rows = M.subsample_rows(10_000)
    want = np.random.Generator(np.random.PCG64(1789)).choice(10_000, size=4096, replace=False)
    assert np.array_equal(rows, want)


def test_metric_record_json_roundtrip(golden):
    from paper_2408_06513_b200.metrics import MetricRecord

    g = golden("metrics")
    for line in g["run_json"]:
        r = MetricRecord.from_json_line(str(line))
        assert r.wall_ms == 0.0
        assert r.to_json_line() == str(line)
        assert list(json.loads(r.to_json_line())) == ["iteration", "binned_stddev", "overplotting",
                                                      "trustworthiness", "ordering"]
