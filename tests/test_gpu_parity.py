"""GPU parity: the CUDA path (through the drop-in API / C ABI) against the oracle and the
golden vectors recorded from the reference.

Tolerances (SURVEY.md section 8(c), fp32 device arithmetic):
  counts                         bit-exact for identical coordinates
  smoothing                      |err| <= 2e-6 * max(values)  (fp32 taps, fp32 accumulation)
  tables                         max |err| / C <= 1e-6; partition identities <= 1e-6 * C
  field                          max |err| <= 1e-6 (field from identical fp32 density)
  constant-density fixed point   <= 1e-6
  positions after T iterations   max |err| <= 2e-5
"""

import numpy as np
import pytest

from conftest import blob, clusters, f32

pytestmark = pytest.mark.gpu

TABLE_TOL = 1e-6
FIELD_TOL = 1e-6
POS_TOL = 2e-5


def maxerr(a, b):
    return float(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)).max())


# ------------------------------------------------------------------------ splat
@pytest.mark.parametrize("k", [1, 3, 6, 8, 10, 12])
def test_accumulate_bit_exact(P, oracle, rng, k):
    pts = np.concatenate([f32(rng.random((20000, 2))), clusters(30000, k),
                          np.array([[0, 0], [1, 1], [1, 0], [0, 1], [0.5, 0.5]], dtype=np.float64)])
    assert np.array_equal(P.accumulate(pts, k), oracle.accumulate(pts, k))


def test_accumulate_float64_inputs_bit_exact(P, oracle, rng):
    pts = rng.random((50000, 2))  # not fp32-representable: binned in float64 on the device
    assert np.array_equal(P.accumulate(pts, 10), oracle.accumulate(pts, 10))


def test_accumulate_golden_and_edges(P, golden):
    g = golden("accumulate")
    assert np.array_equal(P.accumulate(g["positions"], 6), g["counts"])
    assert np.array_equal(P.accumulate(g["positions"], 9), g["counts_k9"])
    assert P.accumulate(np.empty((0, 2)), 3).sum() == 0
    grid = P.accumulate(np.array([[0.3, 0.3]] * 3), 3)
    assert grid[2, 2] == 3 and grid.sum() == 3


def test_splat_hot_pixel_contention(P, oracle):
    pts = np.full((1_000_003, 2), 0.5)
    pts[::7] = 0.25
    assert np.array_equal(P.accumulate(pts, 8), oracle.accumulate(pts, 8))


def test_splat_device_f32_path_bit_exact(P, oracle):
    """The fp32 splat used inside the run loop (inim_splat with float32 points)."""
    import torch
    from paper_2408_06513_b200 import _device as D, _lib

    pts = clusters(1_000_001, 5)
    lib = _lib.load()
    dev = torch.from_numpy(pts.astype(np.float32)).cuda()
    counts = torch.zeros((1024, 1024), dtype=torch.int32, device="cuda")
    _lib.check(lib.inim_splat(D.ptr(dev), 0, len(pts), 10, D.ptr(counts), D.stream()), "splat")
    assert np.array_equal(counts.cpu().numpy().astype(np.float64), oracle.accumulate(pts, 10))


# -------------------------------------------------------------------- smoothing
@pytest.mark.parametrize("s,ks", [(8, 3), (16, 8), (32, 2), (32, 8), (64, 1), (128, 4), (256, 8), (1024, 8),
                                  (512, 16), (64, 5)])
def test_gaussian_smooth_vs_oracle(P, oracle, rng, s, ks):
    g = f32(rng.random((s, s)) ** 3 * 50)
    want = oracle.gaussian_smooth(g, ks)
    got = P.gaussian_smooth(g, ks)
    assert maxerr(got, want) <= 2e-6 * np.abs(want).max()


def test_gaussian_smooth_golden_and_mass(P, golden):
    g = golden("smooth")
    for grid, ks, key in (("g32", 2, "s32_ks2"), ("g32", 8, "s32_ks8"), ("g16", 8, "s16_ks8"), ("g8", 3, "s8_ks3")):
        assert maxerr(P.gaussian_smooth(g[grid], ks), g[key]) <= 2e-6 * np.abs(g[key]).max()
    imp = np.zeros((64, 64))
    imp[0, 0] = 1.0
    assert abs(P.gaussian_smooth(imp, 2).sum() - 1.0) < 1e-5
    with pytest.raises(ValueError):
        P.gaussian_smooth(imp, 0)


@pytest.mark.parametrize("k,ks", [(6, 4), (8, 8), (10, 8)])
def test_build_density_vs_oracle(P, oracle, k, ks):
    pts = clusters(200_000, k)
    tex = P.build_density(pts, P.RegularizationParams(k=k, kernel_size=ks))
    want, bg = oracle.build_density(pts, k, ks)
    assert tex.background == bg
    assert maxerr(tex.values, want) <= 2e-6 * want.max()


def test_build_density_golden_and_errors(P, golden):
    g = golden("density")
    tex = P.build_density(g["positions"], P.RegularizationParams(k=6, kernel_size=4))
    assert maxerr(tex.values, g["values_k6_ks4"]) <= 2e-6 * g["values_k6_ks4"].max()
    tex = P.build_density(np.empty((0, 2)), P.RegularizationParams(k=4, background=1.0))
    assert np.allclose(tex.values, 1.0)
    with pytest.raises(P.ZeroBackground):
        P.build_density(np.empty((0, 2)), P.RegularizationParams(k=4, background=0.0))


# ----------------------------------------------------------------- integral set
@pytest.mark.parametrize("s", [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048])
def test_integral_set_vs_oracle(P, oracle, rng, s):
    d = f32(rng.random((s, s)) * rng.uniform(0.5, 20))
    t = P.build_integral_set(d)
    want, total = oracle.build_integral_set(d)
    assert abs(t.total - total) <= 1e-6 * total
    got = np.stack(t.tables())
    assert maxerr(got, want) / total <= TABLE_TOL


def test_integral_set_golden(P, golden):
    g = golden("integral")
    for s in (2, 4, 8, 16, 32, 64, 128):
        t = P.build_integral_set(g[f"d{s}"])
        assert maxerr(np.stack(t.tables()), g[f"t{s}"]) / g[f"total{s}"] <= TABLE_TOL
    t = P.build_integral_set(g["dint"])
    assert maxerr(np.stack(t.tables()), g["tint"]) / g["totalint"] <= TABLE_TOL


def test_integral_known_answers(P):
    t = P.build_integral_set(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert t.rect_tl[1, 1] == 10 and t.rect_tl[0, 0] == 1
    assert t.rect_bl[0, 0] == 3 and t.rect_tr[0, 0] == 2 and t.rect_br[0, 0] == 4
    t = P.build_integral_set(np.ones((4, 4)))
    assert t.wedge_up[1, 1] == 4.0
    d = np.zeros((8, 8))
    d[2, 6] = 1.0
    t = P.build_integral_set(d)
    assert t.wedge_up[2, 6] == 1.0 and t.wedge_down[2, 6] == 0.0
    with pytest.raises(ValueError):
        P.build_integral_set(np.ones((6, 6)))


def test_integral_counter_and_partitions(P, rng):
    P.scan_counter.reset()
    d = rng.random((16, 16))
    cols = P.column_integrals(d)
    assert P.scan_counter.steps == 2 * 4
    P.scan_counter.reset()
    P.classical_rects(cols)
    assert P.scan_counter.steps == 4 * 4
    P.scan_counter.reset()
    tri = P.triangle_integrals(cols)
    assert P.scan_counter.steps == 4 * 4
    P.scan_counter.reset()
    P.tilted_wedges(tri, cols)
    assert P.scan_counter.steps == 2 * 4
    t = P.build_integral_set(f32(rng.random((256, 256)) * 10))
    rect = t.rect_tl + t.rect_bl + t.rect_br + t.rect_tr
    wedge = t.wedge_up + t.wedge_left + t.wedge_down + t.wedge_right
    assert np.abs(rect - t.total).max() / t.total <= TABLE_TOL
    assert np.abs(wedge - t.total).max() / t.total <= TABLE_TOL


def test_staged_api_vs_oracle(P, oracle, rng):
    d = f32(rng.random((64, 64)) * 5)
    want, total = oracle.build_integral_set(d)
    cols = P.column_integrals(d)
    up, lo = oracle.column_integrals(d)
    assert maxerr(cols.upper, up) <= 1e-6 * total and maxerr(cols.lower, lo) <= 1e-6 * total
    tl, bl, br, tr = P.classical_rects(cols)
    assert maxerr(np.stack([tl, bl, br, tr]), want[:4]) <= 1e-6 * total
    tri = P.triangle_integrals(cols)
    wu, wl, wd, wr = P.tilted_wedges(tri, cols)
    assert maxerr(np.stack([wu, wl, wd, wr]), want[4:]) <= 1e-6 * total


def test_integral_large_sizes_properties(P, rng):
    """4096^2 (BASELINE configs[2] grid): partition identities and spot checks against
    brute-force region sums at sampled pixels."""
    s = 4096
    d = f32(rng.random((s, s)) * 3 + 0.1)
    t = P.build_integral_set(d)
    C = t.total
    assert abs(C - d.sum()) <= 1e-6 * C
    T = np.stack(t.tables())
    assert np.abs(T[:4].sum(0) - C).max() / C <= TABLE_TOL
    assert np.abs(T[4:].sum(0) - C).max() / C <= TABLE_TOL
    jj = np.arange(s)[:, None]
    ii = np.arange(s)[None, :]
    for (j, i) in [(0, 0), (17, 4000), (2048, 2047), (4095, 4095), (1234, 3), (4000, 100)]:
        a, b = ii <= i, jj <= j
        u, w = (ii + jj) <= i + j, (ii - jj) >= i - j
        want = [d[a & b].sum(), d[a & ~b].sum(), d[~a & ~b].sum(), d[~a & b].sum(),
                d[u & w].sum(), d[u & ~w].sum(), d[~u & ~w].sum(), d[~u & w].sum()]
        assert np.abs(T[:, j, i] - want).max() / C <= TABLE_TOL, (j, i)


# -------------------------------------------------------------------- mapping
def test_flat_response_matches_reference(P, golden):
    P.flat_response.clear()
    g = golden("flat")
    for k in (1, 2, 3, 4, 5, 6, 8):
        assert maxerr(P.flat_response.get(k), g[f"defect_k{k}"]) <= 1e-15
    P.flat_response.get(4)
    assert P.flat_response.builds == 7


def test_anchors_known_points(P):
    a = P.anchors(0.5, 0.25)
    assert np.allclose(a.down_right, (1.0, 0.75)) and np.allclose(a.up_left, (0.25, 0.0))
    assert np.allclose(a.up_right, (0.75, 0.0)) and np.allclose(a.down_left, (0.0, 0.75))
    a = P.anchors(0.5, 0.5)
    assert np.allclose(a.down_right, (1, 1)) and np.allclose(a.up_right, (1, 0)) and np.allclose(a.down_left, (0, 1))


def test_raw_and_corrected_map(P, oracle, rng):
    d = f32(rng.random((16, 16)))
    t = P.build_integral_set(d)
    want_t, total = oracle.build_integral_set(d)
    x = y = 0.53
    i = j = 8
    got = P.raw_map(x, y, t)
    A = P.anchors(x, y)
    W = want_t[:, j, i]
    num = (W[0] * A.down_right + W[1] * A.up_right + W[2] * A.up_left + W[3] * A.down_left
           + W[4] * np.array([x, 1.0]) + W[5] * np.array([1.0, y]) + W[6] * np.array([x, 0.0])
           + W[7] * np.array([0.0, y]))
    assert maxerr(got, num / (2 * total)) <= 1e-6
    with pytest.raises(P.SingularMass):
        P.raw_map(0.5, 0.5, P.build_integral_set(np.zeros((4, 4))))
    tc = P.build_integral_set(np.full((64, 64), 2.0))
    X, Y = P.unit_coordinates(6)
    out = P.corrected_map(X, Y, tc, P.flat_response.get(6))
    assert np.abs(out - np.stack([X, Y], -1)).max() <= 1e-6


def test_build_field_vs_oracle_and_golden(P, oracle, golden):
    g = golden("field")
    tables = g["tables"]
    t = P.IntegralSet(*tables, total=float(g["total"]), k=6)
    f = P.build_field(t)
    assert maxerr(f.targets, g["targets"]) <= FIELD_TOL
    assert abs(f.max_excursion - float(g["max_excursion"])) <= FIELD_TOL
    # fused path (density -> field, tables stay on chip) against the oracle on the same fp32 density
    for k, ks in ((6, 4), (8, 8), (10, 8)):
        pts = clusters(100_000, 3 + k)
        tex = P.build_density(pts, P.RegularizationParams(k=k, kernel_size=ks))
        dens = tex.values  # the device density (fp32 values), fed identically to the oracle
        t8, total = oracle.build_integral_set(dens)
        want, wexc = oracle.build_field(t8, total, k)
        new, fld, _ = P.iterate_once(pts, P.RegularizationParams(k=k, kernel_size=ks))
        assert maxerr(fld.targets, want) <= FIELD_TOL, k
        assert abs(fld.max_excursion - wexc) <= FIELD_TOL


@pytest.mark.parametrize("k", [5, 6, 8, 10, 12])
def test_fixed_point_constant_density(P, k):
    """SPEC fixed point (test_acceptance.py:91-100): constant density -> identity field."""
    s = 1 << k
    t = P.build_integral_set(np.full((s, s), 1.7))
    f = P.build_field(t)
    X, Y = P.unit_coordinates(k)
    assert np.abs(f.targets - np.stack([X, Y], -1)).max() <= 1e-6


def test_sample_field(P, golden, rng):
    g = golden("sample")
    fld = P.DeformationField(targets=g["targets"], k=4)
    assert maxerr(P.sample_field(fld, g["points"]), g["out"]) <= 1e-15  # float64 field: float64 path
    ident = P.DeformationField(targets=np.stack(P.unit_coordinates(5), -1), k=5)
    pts = rng.random((300, 2))
    pts[:5] = [[0, 0], [1, 1], [1, 0], [0, 1], [0.999999, 0.5]]
    assert np.abs(P.sample_field(ident, pts) - pts).max() < 1e-12
    assert P.interpolate(ident, [0.25, 0.75]).shape == (2,)


# ------------------------------------------------------------- iterate / run
def test_iterate_once_golden(P, golden):
    g = golden("iterate")
    new, fld, dens = P.iterate_once(g["positions"], P.RegularizationParams(k=6, kernel_size=4))
    assert maxerr(dens.values, g["density"]) <= 2e-6 * g["density"].max()
    assert maxerr(fld.targets, g["targets"]) <= FIELD_TOL
    assert maxerr(new, g["new_positions"]) <= FIELD_TOL


def test_run_c1_matches_reference_frames(P, golden):
    """BASELINE configs[0]: 3-cluster 10k points, 256^2, ks=8, 5 iterations."""
    g = golden("run_c1")
    r = P.run(P.ScatterDataset(positions=g["positions"]), P.RegularizationParams(k=8, kernel_size=8, iterations=5))
    assert r.iterations == 5
    for t in range(6):
        assert maxerr(r.frame(t), g["frames"][t]) <= POS_TOL, t
    assert maxerr(r.fields[-1].targets, g["field_last"]) <= 5 * FIELD_TOL


def test_run_displacement_stop_golden(P, golden):
    g = golden("run_disp")
    pr = P.RegularizationParams(k=6, iterations=50, stop="displacement", epsilon=float(g["epsilon"]))
    r = P.run(P.ScatterDataset(positions=g["positions"]), pr)
    assert r.iterations == int(g["n_iters"])
    assert maxerr(r.frame(r.iterations), g["last"]) <= POS_TOL


def test_run_matches_oracle_c2_like(P, oracle):
    """1M points, 1024^2, 3 iterations against the float64 oracle."""
    pts = clusters(1_000_000, 4)
    frames = oracle.run_positions(pts, 10, 8, 3)
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=10, kernel_size=8, iterations=3),
              store_fields=False)
    for t in range(4):
        assert maxerr(r.frame(t), frames[t]) <= POS_TOL, t


def test_run_semantics(P):
    ds = P.ScatterDataset(positions=blob())
    r0 = P.run(ds, P.RegularizationParams(k=6, iterations=0))
    assert r0.iterations == 0 and np.array_equal(r0.frame(0), ds.positions)
    a = P.run(ds, P.RegularizationParams(k=6, iterations=3))
    b = P.run(ds, P.RegularizationParams(k=6, iterations=3))
    for t in range(4):
        assert np.array_equal(a.frame(t), b.frame(t))
    P.flat_response.clear()
    P.run(ds, P.RegularizationParams(k=6, iterations=4))
    assert P.flat_response.builds == 1
    full = P.run(ds, P.RegularizationParams(k=6, iterations=9, frame_cap=64))
    capped = P.run(ds, P.RegularizationParams(k=6, iterations=9, frame_cap=4))
    for t in (3, 5, 7, 9):
        assert np.array_equal(capped.frame(t), full.frame(t))
    rt = P.run(ds, P.RegularizationParams(k=6, iterations=50, stop="time", time_budget=1e-9))
    assert rt.iterations == 0
    r8 = P.run(ds, P.RegularizationParams(k=6, iterations=8))
    assert np.array_equal(P.transition_positions(r8, 0.0), ds.positions)
    assert np.array_equal(P.transition_positions(r8, 8.0), r8.frame(8))
    assert np.allclose(P.transition_positions(r8, 1.5), 0.5 * (r8.frame(1) + r8.frame(2)), atol=0)
    with pytest.raises(P.OutOfRangeLevel):
        P.transition_positions(r8, 8.5)
    r4 = P.run(ds, P.RegularizationParams(k=6, iterations=4))
    assert np.array_equal(P.map_through(r4, ds.positions), r4.frame(4))
    assert np.array_equal(P.map_through(r4, ds.positions, upto=2), r4.frame(2))
    assert len(r4.wall_times) == 4 and all(w > 0 for w in r4.wall_times)


def test_uniform_grid_near_fixed_point(P):
    X, Y = P.unit_coordinates(5)
    pos = np.column_stack([X.ravel(), Y.ravel()])
    new, _f, _d = P.iterate_once(pos, P.RegularizationParams(k=5, kernel_size=2))
    assert np.abs(new - pos).max() < 2e-6


def test_order_preserved_and_cluster_expands(P, rng):
    pts = np.concatenate([np.clip(rng.normal((0.3, 0.5), 0.03, (400, 2)), 0, 1),
                          np.clip(rng.normal((0.7, 0.5), 0.03, (100, 2)), 0, 1)])
    new, _f, _d = P.iterate_once(pts, P.RegularizationParams(k=7, kernel_size=8))
    left, right = new[:400, 0], new[400:, 0]
    assert left.mean() < right.mean() and np.quantile(left, 0.99) < np.quantile(right, 0.01)
    spread0 = np.linalg.norm(pts[:400] - pts[:400].mean(0), axis=1).mean()
    spread1 = np.linalg.norm(new[:400] - new[:400].mean(0), axis=1).mean()
    assert spread1 > spread0


def test_neighbourhood_ordering_preserved(P, oracle):
    """Pairwise x/y order identical for pairs separated by more than 2*tol."""
    pts = clusters(10_000, 9)
    want = oracle.run_positions(pts, 8, 8, 5)[-1]
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=8, kernel_size=8, iterations=5))
    got = r.frame(5)
    sub = np.random.default_rng(1789).choice(len(pts), 1500, replace=False)
    for ax in (0, 1):
        dw = want[sub, ax][:, None] - want[sub, ax][None, :]
        dg = got[sub, ax][:, None] - got[sub, ax][None, :]
        sep = np.abs(dw) > 2 * POS_TOL
        assert np.array_equal(np.sign(dw[sep]), np.sign(dg[sep]))


def test_run_host_abi_end_to_end(P, oracle):
    """inim_run_host: the host-buffer C ABI call (float64 in/out)."""
    import ctypes
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    pts = np.ascontiguousarray(clusters(100_000, 2))
    out = np.empty_like(pts)
    rc = lib.inim_run_host(pts.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), len(pts),
                           8, 8, 0.0, 3)
    assert rc == 0
    want = oracle.run_positions(pts, 8, 8, 3)[-1]
    assert maxerr(out, want) <= POS_TOL


@pytest.mark.parametrize("points,iters,max_batch", [(20_000, 4, 4), (70_000, 4, 3), (30_000, 2, 8)])
def test_splom_batch_matches_single_plot_runs(P, oracle, points, iters, max_batch):
    """A batched SPLOM run (inim_run_batched: plot index in grid.z, the wide 32 x 128
    tile geometry) against each plot regularized alone (the 16 x 64 tiles of a single
    256^2 plot) and against the oracle, within the float32 tolerance; with and without
    the per-run point sort (n >= 65,536 and >= 3 iterations), in chunks of max_batch
    plots; its per-plot frame statistics equal the reference metrics of its own frames,
    and a replay of the captured graph reproduces the run bit for bit."""
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot

    cfg = SplomConfig(nplots=5, points=points, k=8, kernel_size=8, iterations=iters, max_batch=max_batch,
                      collect_metrics=True)
    job = DeviceSplom(cfg, range(cfg.nplots))
    job.load(lambda i: splom_plot(i, cfg.points))
    res = job.run().cpu().numpy().astype(np.float64)
    mets = job.metrics()
    for i in range(cfg.nplots):
        pts = splom_plot(i, cfg.points)
        r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=8, kernel_size=8, iterations=iters),
                  store_fields=False)
        assert maxerr(res[i], r.frame(iters)) <= POS_TOL, i
        assert maxerr(res[i], oracle.run_positions(pts, 8, 8, iters)[-1]) <= POS_TOL, i
        want = (oracle.binned_stddev(res[i], 8), oracle.overplotting(res[i], 8))
        assert mets[i][-1] == pytest.approx(want, rel=1e-12, abs=0), i
    again = job.run().cpu().numpy().astype(np.float64)  # graph replay: same answer
    assert np.array_equal(again, res)
    import torch  # host buffers, chunked copies overlapping the runs: the same answer
    hin = torch.empty(tuple(job.inputs.shape), dtype=torch.float32).pin_memory()
    hin.copy_(job.inputs.cpu())
    hout = torch.empty_like(hin).pin_memory()
    job.run_host(hin, hout, chunk=2)
    torch.cuda.synchronize()
    assert np.array_equal(hout.numpy().astype(np.float64), res)


@pytest.mark.parametrize("k", [11, 12])
def test_larger_grids_run_against_oracle(P, oracle, k):
    """2048^2 and 4096^2 grids (BASELINE configs[2] grid size), 2 iterations."""
    pts = clusters(400_000, k)
    frames = oracle.run_positions(pts, k, 8, 2)
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=k, kernel_size=8, iterations=2),
              store_fields=False)
    for t in range(3):
        assert maxerr(r.frame(t), frames[t]) <= POS_TOL, t


@pytest.mark.parametrize("k", [9, 12])
def test_field_layouts_bit_identical(tmp_path, k):
    """The move's paired (s, s, 4) and plain (s, s, 2) field layouts (INIM_PAIRS; paired
    by default up to 2048^2, plain above) give bit-identical runs: same weights, same
    blend order, only the gathers differ."""
    import os
    import subprocess
    import sys
    import textwrap

    from conftest import ROOT

    host = clusters(120_000, k).astype(np.float32)
    np.save(tmp_path / "in.npy", host)
    outs = []
    for pairs in ("0", "1"):
        dst = tmp_path / f"out{pairs}.npy"
        script = textwrap.dedent(f"""
            import sys
            sys.path.insert(0, {str(ROOT)!r})
            import numpy as np, torch
            from paper_2408_06513_b200 import _device as D, _lib
            lib = _lib.load()
            host = np.load({str(tmp_path / "in.npy")!r})
            n = len(host)
            ws = torch.empty(int(lib.inim_workspace_bytes({k}, n, 1)), dtype=torch.uint8, device="cuda")
            a = torch.from_numpy(host).cuda()
            _lib.check(lib.inim_run_uncached(D.ptr(a), n, {k}, 8, 0.0, 4, 0.0, None, None, None, None, None,
                                             D.ptr(ws), D.stream()), "run")
            np.save({str(dst)!r}, a.cpu().numpy())
        """)
        f = tmp_path / f"layout{pairs}.py"
        f.write_text(script)
        out = subprocess.run([sys.executable, str(f)], capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, INIM_PAIRS=pairs))
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(np.load(dst))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("k,n,ks,metrics", [(10, 200_000, 8, False), (8, 70_000, 8, True), (12, 300_000, 5, False),
                                            (9, 100_000, 20, True)])
def test_float_counts_bit_identical(tmp_path, k, n, ks, metrics):
    """Sorted runs splat with 16-byte float reductions into float32 counts (the default);
    INIM_F32_COUNTS=0 keeps uint32 counts with one reduction per pixel.  Counts are exact
    integers either way, so the runs (and the per-frame statistics) are bit-identical."""
    import os
    import subprocess
    import sys
    import textwrap

    from conftest import ROOT

    host = clusters(n, k).astype(np.float64)
    np.save(tmp_path / "in.npy", host)
    outs = []
    for mode in ("0", "1"):
        dst = tmp_path / f"out{mode}.npz"
        script = textwrap.dedent(f"""
            import sys
            sys.path.insert(0, {str(ROOT)!r})
            import numpy as np
            import paper_2408_06513_b200 as P
            host = np.load({str(tmp_path / "in.npy")!r})
            r = P.run(P.ScatterDataset(positions=host), P.RegularizationParams(k={k}, kernel_size={ks}, iterations=4),
                      collect_metrics={"'basic'" if metrics else "'none'"}, store_fields=False)
            m = np.array([[x.binned_stddev, x.overplotting] for x in r.metrics]) if r.metrics else np.zeros((0, 2))
            np.savez({str(dst)!r}, pos=r.frame(4), m=m)
        """)
        f = tmp_path / f"fc{mode}.py"
        f.write_text(script)
        out = subprocess.run([sys.executable, str(f)], capture_output=True, text=True, timeout=300,
                             env=dict(os.environ, INIM_F32_COUNTS=mode))
        assert out.returncode == 0, out.stderr[-2000:]
        outs.append(np.load(dst))
    assert np.array_equal(outs[0]["pos"], outs[1]["pos"])
    assert np.array_equal(outs[0]["m"], outs[1]["m"])


def test_splom_batch_displacement_stop(P, oracle):
    """stop="displacement" in a batched run: each plot stops after its own iteration
    whose max |delta| < epsilon (regularize.py:76-79) while the rest of the batch goes on;
    iteration counts and final positions match one run per plot and the oracle."""
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot

    eps = 0.019  # the oracle's displacements cross it at iterations 9, 9, 9, 10 (margins >= 6e-4)
    cfg = SplomConfig(nplots=4, points=20_000, k=8, kernel_size=8, iterations=30, stop="displacement", epsilon=eps,
                      collect_metrics=True)
    job = DeviceSplom(cfg, range(cfg.nplots))
    job.load(lambda i: splom_plot(i, cfg.points))
    res = job.run().cpu().numpy().astype(np.float64)
    done = job.iterations_done()
    mets = job.metrics()
    assert len(set(done)) > 1, done  # the plots stop at different iterations
    for i in range(cfg.nplots):
        pts = splom_plot(i, cfg.points)
        r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=8, kernel_size=8, iterations=30,
                                                                          stop="displacement", epsilon=eps))
        frames = oracle.run_positions(pts, 8, 8, 30, stop="displacement", epsilon=eps)
        assert done[i] == r.iterations == len(frames) - 1, (i, done[i], r.iterations, len(frames) - 1)
        assert maxerr(res[i], r.frame(r.iterations)) <= POS_TOL, i
        assert maxerr(res[i], frames[-1]) <= POS_TOL, i
        assert len(mets[i]) == done[i]
