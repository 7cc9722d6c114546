"""GPU parity of the layout metrics (metrics.py:46-168) through the drop-in API and the
C ABI (inim_frame_stats / inim_trust_penalty / inim_order_pairs / inim_run_metrics).

Bars: occupied-pixel counts, trustworthiness penalty sums and preserved-pair counts are
integers and must be identical to the oracle's (hence overplotting, trustworthiness and
ordering bit-identical); binned_stddev is the same correctly-rounded function of exact
integer moments (identical), and within 1e-12 relative of the reference's numpy std.
Run records are checked against the oracle applied to the run's OWN frames (exact), and
against the reference's records (golden) within the position tolerance's effect.
"""

import numpy as np
import pytest

from conftest import blob, clusters, f32

pytestmark = pytest.mark.gpu

STD_REL = 1e-12


@pytest.mark.parametrize("k", [0, 1, 2, 3, 6, 8, 10, 12])
def test_frame_stats_match_oracle(P, oracle, rng, k):
    from paper_2408_06513_b200 import metrics as M

    pts = np.concatenate([f32(rng.random((20000, 2))), clusters(30000, k + 1), f32(np.array([[0, 0], [1, 1]]))])
    assert M.frame_stats(pts, k) == oracle.frame_stats(pts, k)[:2] + (len(pts),)
    if k >= 2:
        assert P.binned_stddev(pts, k) == oracle.binned_stddev(pts, k)
    assert P.overplotting(pts, k) == oracle.overplotting(pts, k)


def test_occupancy_golden(P, golden):
    g = golden("metrics")
    for k in (2, 4, 6, 8):
        pts = g[f"occ_pts_k{k}"]
        assert P.overplotting(pts, k) == g[f"occ_over_k{k}"]
        assert P.binned_stddev(pts, k) == pytest.approx(float(g[f"occ_binned_k{k}"]), rel=STD_REL, abs=0)
    assert P.binned_stddev(g["occ_uniform"], 4) == 0.0
    assert P.overplotting(g["occ_uniform"], 4) == 0.0


def test_occupancy_edge_cases(P):
    with pytest.raises(ValueError):
        P.binned_stddev(np.zeros((3, 2)), 1)
    assert P.binned_stddev(np.empty((0, 2)), 4) == 0.0
    with pytest.raises(P.EmptyDataset):
        P.overplotting(np.empty((0, 2)), 4)
    assert P.overplotting(np.full((10, 2), 0.5), 4) == 0.9


def test_neighbourhood_golden(P, golden):
    g = golden("metrics")
    o, m = g["nb_orig"], g["nb_moved"]
    assert P.trustworthiness(o, m, 10) == g["nb_trust10"]
    assert P.trustworthiness(o, m, 3) == g["nb_trust3"]
    assert P.orthogonal_ordering(o, m) == g["nb_order"]
    assert P.trustworthiness(o, o) == 1.0 and P.orthogonal_ordering(o, o) == 1.0
    assert P.orthogonal_ordering(g["nb_big"], g["nb_bigm"]) == g["nb_order_big"]
    assert P.orthogonal_ordering(g["nb_big"], g["nb_bigm"], 1000) == g["nb_order_big_cap"]


@pytest.mark.parametrize("n,nn", [(11, 10), (257, 1), (1000, 10), (4096, 10), (3000, 50)])
def test_neighbourhood_match_oracle(P, oracle, rng, n, nn):
    o = f32(rng.random((n, 2)))
    o[5:9] = o[0]  # exact ties: broken toward the lower index
    m = f32(np.clip(o + rng.normal(0, 0.03, o.shape), 0, 1))
    assert P.trustworthiness(o, m, nn) == oracle.trustworthiness(o, m, nn)
    assert P.orthogonal_ordering(o, m) == oracle.orthogonal_ordering(o, m)


def test_neighbourhood_errors(P):
    with pytest.raises(ValueError):
        P.trustworthiness(np.zeros((20, 2)), np.zeros((21, 2)))
    with pytest.raises(P.TooFewSamples):
        P.trustworthiness(np.zeros((10, 2)), np.zeros((10, 2)), 10)
    with pytest.raises(ValueError):
        P.orthogonal_ordering(np.zeros((20, 2)), np.zeros((21, 2)))
    assert P.orthogonal_ordering(np.zeros((1, 2)), np.zeros((1, 2))) == 1.0


def _check_records_against_own_frames(oracle, r, original, k, full, nn=10):
    assert len(r.metrics) == r.iterations + 1
    for t, rec in enumerate(r.metrics):
        assert rec.iteration == t
        b, o, tr, od = oracle.record_for_frame(original, r.frame(t), k, full=full, n_neighbors=nn)
        assert rec.binned_stddev == pytest.approx(b, rel=STD_REL, abs=0)
        assert rec.overplotting == o
        assert rec.trustworthiness == tr
        assert rec.ordering == od
        assert rec.wall_ms >= 0.0


def test_run_full_metrics_golden(P, oracle, golden):
    """run(collect_metrics='full') on the reference's C1 layout (10k points, 4096-row
    subsample): exact against the oracle on our frames; frame 0 exact against the
    reference; later frames within what the 2e-5 position tolerance allows."""
    g = golden("metrics")
    pts, k = g["run_positions"], int(g["run_k"])
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=k, kernel_size=8, iterations=3),
              collect_metrics="full")
    _check_records_against_own_frames(oracle, r, pts, k, True)
    rec0 = r.metrics[0]
    assert rec0.binned_stddev == pytest.approx(float(g["run_binned"][0]), rel=STD_REL, abs=0)
    assert (rec0.overplotting, rec0.trustworthiness, rec0.ordering) == (g["run_over"][0], 1.0, 1.0)
    for t in range(1, 4):
        rec = r.metrics[t]
        assert rec.binned_stddev == pytest.approx(float(g["run_binned"][t]), rel=2e-3)
        assert abs(rec.overplotting - g["run_over"][t]) <= 2e-3
        assert abs(rec.trustworthiness - g["run_trust"][t]) <= 1e-3
        assert abs(rec.ordering - g["run_order"][t]) <= 1e-3


def test_run_basic_metrics_sorted_path(P, oracle):
    """>= 65536 points: the run sorts the points by pixel; the per-frame statistics come
    off the counts the moves splat, the subsample through the sort permutation."""
    pts = clusters(150_000, 5)
    k = 9
    for mode in ("basic", "full"):
        r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=k, kernel_size=8, iterations=4),
                  collect_metrics=mode, store_fields=False)
        _check_records_against_own_frames(oracle, r, pts, k, mode == "full")
        if mode == "basic":
            assert all(rec.trustworthiness is None and rec.ordering is None for rec in r.metrics)


def test_run_metrics_chunks_and_stops(P, oracle):
    pts = blob(3000)
    # more iterations than one captured chunk (16) and frame thinning
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=6, kernel_size=4, iterations=20, frame_cap=4),
              collect_metrics="basic")
    assert [m.iteration for m in r.metrics] == list(range(21))
    for t in (0, 7, 13, 20):
        b, o, _, _ = oracle.record_for_frame(pts, r.frame(t), 6)
        assert r.metrics[t].binned_stddev == pytest.approx(b, rel=STD_REL, abs=0)
        assert r.metrics[t].overplotting == o
    # displacement stop: one record per executed iteration
    rd = P.run(P.ScatterDataset(positions=pts),
               P.RegularizationParams(k=6, iterations=50, stop="displacement", epsilon=5e-3), collect_metrics="full")
    assert len(rd.metrics) == rd.iterations + 1 < 51
    _check_records_against_own_frames(oracle, rd, pts, 6, True)
    # time budget: iterations launched one by one
    rt = P.run(P.ScatterDataset(positions=pts),
               P.RegularizationParams(k=6, iterations=3, stop="time", time_budget=60.0), collect_metrics="full")
    _check_records_against_own_frames(oracle, rt, pts, 6, True)


def test_run_metrics_small_and_empty(P):
    few = f32(np.array([[0.1, 0.2], [0.5, 0.5], [0.9, 0.3]]))
    r = P.run(P.ScatterDataset(positions=few), P.RegularizationParams(k=4, iterations=2), collect_metrics="full")
    assert len(r.metrics) == 3 and all(m.trustworthiness is None for m in r.metrics)
    e = P.run(P.ScatterDataset(positions=np.empty((0, 2))), P.RegularizationParams(k=4, iterations=2),
              collect_metrics="basic")
    assert [(m.binned_stddev, m.overplotting) for m in e.metrics] == [(0.0, 0.0)] * 3


def test_frame_stats_abi_symbols(P):
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    for name in ("inim_frame_stats", "inim_trust_penalty", "inim_order_pairs", "inim_gather_points",
                 "inim_run_metrics"):
        assert hasattr(lib, name)
