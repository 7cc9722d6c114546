"""GPU parity at the shapes the benchmark numbers are quoted on (BASELINE.json configs,
SURVEY.md section 8(c)/(d)), plus the functional range the reference accepts.

  C2  bench.py's own four-cluster 1M input, 1024^2, all 10 iterations vs the oracle;
      neighbourhood ordering: pairwise x/y order of the fixed-seed 4096 subsample and
      10-NN set agreement >= 99.9% (metrics.py:74-87, 132-134)
  C3  bench.py's 16M gaussian-mixture input, 4096^2, 10 iterations vs the oracle
  C4  SPLOM plots (500k points, 1024^2, 10 iterations) vs the oracle
  C5  8192^2 and 16384^2 tables (and 32768^2, the device path's largest grid):
      partition identities on the whole grid and brute-force region sums at
      corner / edge / diagonal pixels
  kernel_size > 16 (generic-tap smoothing, density.py:30-51), including kernels longer
  than the reflection period

Brute-force region sums are evaluated on the device in float64 from a row prefix of d
(the region definitions of integral.py:180-228 / model.py:59-85), the checker for grids
whose float64 tables do not fit the host.
"""

import numpy as np
import pytest

from conftest import clusters, f32

pytestmark = pytest.mark.gpu

POS_TOL = 2e-5
TABLE_TOL = 1e-6
FIELD_TOL = 1e-6


def maxerr(a, b):
    return float(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)).max())


def bench_module():
    import bench

    return bench


@pytest.fixture(scope="module")
def oracle_mt(oracle):
    import os

    oracle.set_threads(os.cpu_count() or 1)
    return oracle


def oracle_frames(oracle, pts, k, ks, iters, keep):
    """Frames `keep` of the oracle run (regularize.run's numeric path, float64)."""
    defect = oracle.flat_response(k)
    out = {0: pts} if 0 in keep else {}
    pos = pts
    for t in range(1, iters + 1):
        pos = oracle.iterate_once(pos, k, ks, None, defect)
        if t in keep:
            out[t] = pos
    return out


# ------------------------------------------------------------- neighbourhood ordering
def subsample_rows(n, cap=4096):
    """The fixed-seed pick of metrics.py:132-134 (PCG64 seed 1789)."""
    return np.random.Generator(np.random.PCG64(1789)).choice(n, size=cap, replace=False)


def knn_sets(p, nn=10):
    d = ((p[:, None, :] - p[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d, np.inf)
    idx = np.argpartition(d, nn, axis=1)[:, :nn]
    return [frozenset(r) for r in idx.tolist()]


def assert_neighbourhoods(got, want, tol=POS_TOL):
    """pairwise x- and y-order identical for every pair whose reference
    separation exceeds 2 tol; 10-NN sets identical for >= 99.9% of the subsample."""
    rows = subsample_rows(len(want))
    g, w = got[rows], want[rows]
    for ax in (0, 1):
        dw = w[:, None, ax] - w[None, :, ax]
        dg = g[:, None, ax] - g[None, :, ax]
        sep = np.abs(dw) > 2 * tol
        assert np.all(np.sign(dg[sep]) == np.sign(dw[sep])), ax
    a, b = knn_sets(g), knn_sets(w)
    agree = sum(x == y for x, y in zip(a, b)) / len(a)
    assert agree >= 0.999, agree


# ------------------------------------------------------------------------------ C2
def test_c2_bench_input_all_iterations(P, oracle_mt):
    """bench.py's timed workload: four_cluster(1M, seed=4), k=10, ks=8, 10 iterations."""
    B = bench_module()
    pts = B.four_cluster(B.N_POINTS, seed=4)
    want = oracle_frames(oracle_mt, pts, 10, 8, 10, set(range(11)))
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=10, kernel_size=8, iterations=10),
              store_fields=False)
    assert r.iterations == 10
    for t in range(11):
        assert maxerr(r.frame(t), want[t]) <= POS_TOL, t
    assert_neighbourhoods(r.frame(10), want[10])


# ------------------------------------------------------------------------------ C3
def test_c3_bench_input_ten_iterations(P, oracle_mt):
    """bench.py --workload c3: 16M gaussian-mixture points, 4096^2, 10 iterations."""
    B = bench_module()
    pts = B.c3_points(16_000_000, seed=42)
    keep = {1, 3, 10}
    want = oracle_frames(oracle_mt, pts, 12, 8, 10, keep)
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=12, kernel_size=8, iterations=10),
              store_fields=False)
    for t in sorted(keep):
        assert maxerr(r.frame(t), want[t]) <= POS_TOL, t
    assert_neighbourhoods(r.frame(10), want[10])


# ------------------------------------------------------------------------------ C4
def test_c4_splom_batch_against_oracle(P, oracle_mt):
    """BASELINE configs[3] plot shape through the batched SPLOM path: 3 plots of 500k
    points, 1024^2, 10 iterations, one batched run, each plot against the oracle."""
    from paper_2408_06513_b200.splom import DeviceSplom, SplomConfig, splom_plot

    cfg = SplomConfig(nplots=3, points=500_000, k=10, kernel_size=8, iterations=10)
    job = DeviceSplom(cfg, range(cfg.nplots))
    job.load(lambda i: splom_plot(i, cfg.points))
    res = job.run().cpu().numpy().astype(np.float64)
    for i in range(cfg.nplots):
        want = oracle_frames(oracle_mt, splom_plot(i, cfg.points), 10, 8, 10, {10})
        assert maxerr(res[i], want[10]) <= POS_TOL, i


# ------------------------------------------------------------------------------ C5
class DeviceBrute:
    """Region sums of d at single pixels, float64 on the device: per row j', the
    columns of each region form one interval, summed from the row prefix P."""

    def __init__(self, d):
        import torch

        self.torch = torch
        self.s = d.shape[0]
        self.P = torch.cumsum(d.to(torch.float64), dim=1)

    def _rows(self, lo, hi):
        """sum over rows j' of d[j', lo[j']..hi[j']] (inclusive, clipped; empty if lo > hi)."""
        torch, s, P = self.torch, self.s, self.P
        lo = lo.clamp(0, s)
        hi = hi.clamp(-1, s - 1)
        ok = lo <= hi
        hi_c = hi.clamp(min=0)
        top = P.gather(1, hi_c[:, None])[:, 0]
        low = torch.where(lo > 0, P.gather(1, (lo - 1).clamp(min=0)[:, None])[:, 0], torch.zeros_like(top))
        return float(torch.where(ok, top - low, torch.zeros_like(top)).sum())

    def tables_at(self, j, i):
        torch, s = self.torch, self.s
        jr = torch.arange(s, device=self.P.device, dtype=torch.int64)
        big = torch.full_like(jr, s)
        zero = torch.zeros_like(jr)
        above = jr <= j
        ii = torch.full_like(jr, i)
        # rect: rows <= j / > j, columns <= i / > i
        tl = self._rows(zero, torch.where(above, ii, -ii - 1))
        bl = self._rows(zero, torch.where(~above, ii, -ii - 1))
        br = self._rows(torch.where(~above, ii + 1, big), big)
        tr = self._rows(torch.where(above, ii + 1, big), big)
        u = i + j - jr   # i' <= u  <=>  i' + j' <= i + j
        w = i - j + jr   # i' >= w  <=>  i' - j' >= i - j
        up = self._rows(w, u)
        left = self._rows(zero, torch.minimum(u, w - 1))
        down = self._rows(u + 1, w - 1)
        right = self._rows(torch.maximum(u + 1, w), big)
        return np.array([tl, bl, br, tr, up, left, down, right])


def ones_tables_at(s, j, i):
    """The same region pixel counts for a constant texture (closed per-row lengths)."""
    jr = np.arange(s, dtype=np.int64)

    def rows(lo, hi):
        lo = np.maximum(lo, 0)
        hi = np.minimum(hi, s - 1)
        return float(np.maximum(hi - lo + 1, 0).sum())

    above = jr <= j
    zero, big = np.zeros_like(jr), np.full_like(jr, s)
    ii = np.full_like(jr, i)
    u, w = i + j - jr, i - j + jr
    return np.array([rows(zero, np.where(above, ii, -1)), rows(zero, np.where(~above, ii, -1)),
                     rows(np.where(~above, ii + 1, big), big), rows(np.where(above, ii + 1, big), big),
                     rows(w, u), rows(zero, np.minimum(u, w - 1)), rows(u + 1, w - 1),
                     rows(np.maximum(u + 1, w), big)])


def raw_map_at(t8, C, x, y):
    """_weighted_components (mapping.py:64-77) at one pixel coordinate, float64."""
    below, near = y < x, x + y < 1.0
    drx, dry = (1.0, 1.0 + y - x) if below else (1.0 - y + x, 1.0)
    ulx, uly = (x - y, 0.0) if below else (0.0, y - x)
    urx, ury = (x + y, 0.0) if near else (1.0, x + y - 1.0)
    dlx, dly = (0.0, x + y) if near else (x + y - 1.0, 1.0)
    tl, bl, br, tr, up, left, down, right = t8
    inv = 0.5 / C
    tx = (tl * drx + bl * urx + br * ulx + tr * dlx + (up + down) * x + left) * inv
    ty = (tl * dry + bl * ury + br * uly + tr * dly + (left + right) * y + up) * inv
    return np.array([tx, ty])


def spot_pixels(s):
    h = s // 2
    return [(0, 0), (0, s - 1), (s - 1, 0), (s - 1, s - 1), (h, h), (h - 1, h), (h, h - 1), (17, s - 4),
            (s - 3, 5), (s // 3, s // 3), (s // 5, s - 1 - s // 5), (s - 1, s // 7), (s // 7, s - 1),
            (1, 1), (s - 2, s - 2), (3, s - 2), (s // 3 + 1, 2 * s // 3), (s - 1, h), (h, 0), (1234 % s, 77 % s)]


def device_tables(P, d, k):
    import torch
    from paper_2408_06513_b200 import _device as D, _lib

    lib = _lib.load()
    s = 1 << k
    tables = torch.empty((8, s, s), dtype=torch.float32, device=d.device)
    total = torch.empty(1, dtype=torch.float64, device=d.device)
    ws = torch.empty(int(lib.inim_workspace_bytes(k, 0, 1)), dtype=torch.uint8, device=d.device)
    _lib.check(lib.inim_integral_set(D.ptr(d), k, D.ptr(tables), D.ptr(total), D.ptr(ws), D.stream()), "integral")
    del ws
    return tables, float(total.item())


def c5_texture(k, device):
    """rng.random((s, s)) * rng.uniform(0.5, 20), PCG64 seed 1234 (the
    test_acceptance.py:60-66 pattern), fp32."""
    import torch

    s = 1 << k
    if k <= 14:
        rng = np.random.Generator(np.random.PCG64(1234))
        host = (rng.random((s, s)) * rng.uniform(0.5, 20)).astype(np.float32)
        return torch.from_numpy(host).to(device)
    g = torch.Generator(device=device)
    g.manual_seed(1234)
    return torch.rand((s, s), generator=g, device=device, dtype=torch.float32) * 7.5


def check_partitions(tables, C):
    import torch

    s = tables.shape[1]
    worst = 0.0
    for r0 in range(0, s, 1024):
        blk = tables[:, r0:r0 + 1024].to(torch.float64)
        worst = max(worst, float((blk[:4].sum(0) - C).abs().max()), float((blk[4:].sum(0) - C).abs().max()))
    assert worst / C <= TABLE_TOL, worst / C


@pytest.mark.parametrize("k", [13, 14, 15])
def test_c5_tables_large_grids(P, k):
    """8192^2, 16384^2 (BASELINE configs[4]) and 32768^2: total, partition identities
    over the whole grid, eight tables at 20 corner / edge / diagonal pixels."""
    import torch

    d = c5_texture(k, "cuda")
    s = 1 << k
    tables, C = device_tables(P, d, k)
    ref_total = float(d.to(torch.float64).sum())
    assert abs(C - ref_total) <= 1e-9 * ref_total
    check_partitions(tables, C)
    brute = DeviceBrute(d)
    for (j, i) in spot_pixels(s):
        got = tables[:, j, i].to(torch.float64).cpu().numpy()
        want = brute.tables_at(j, i)
        assert np.abs(got - want).max() / C <= TABLE_TOL, (j, i, got, want)


@pytest.mark.parametrize("k", [14, 15])
def test_field_large_grids_at_spot_pixels(P, k):
    """build_field fused with the integral pass (inim_field_from_density) at 16384^2
    and 32768^2: targets at spot pixels = clip((x, y) + raw(tables) - raw(flat)) from
    brute-force region sums (mapping.py:146-204)."""
    import torch
    from paper_2408_06513_b200 import _device as D, _lib

    lib = _lib.load()
    s = 1 << k
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    # a smooth non-uniform density: a ramp plus noise, so the field moves
    jj = torch.arange(s, device="cuda", dtype=torch.float32)[:, None] / s
    d = (1.0 + 2.0 * jj + 0.5 * torch.rand((s, s), generator=g, device="cuda")).contiguous()
    targets = torch.empty((s, s, 2), dtype=torch.float32, device="cuda")
    exc = torch.zeros(1, dtype=torch.float32, device="cuda")
    total = torch.empty(1, dtype=torch.float64, device="cuda")
    ws = torch.empty(int(lib.inim_workspace_bytes(k, 0, 1)), dtype=torch.uint8, device="cuda")
    _lib.check(lib.inim_field_from_density(D.ptr(d), k, None, D.ptr(targets), D.ptr(exc), D.ptr(total), D.ptr(ws),
                                           D.stream()), "field")
    del ws
    C = float(total.item())
    brute = DeviceBrute(d)
    flat_C = float(s) * s
    for (j, i) in spot_pixels(s):
        x, y = i / s, j / s
        raw = raw_map_at(brute.tables_at(j, i), C, x, y)
        flat = raw_map_at(ones_tables_at(s, j, i), flat_C, x, y)
        want = np.clip(np.array([x, y]) + raw - flat, 0.0, 1.0)
        got = targets[j, i].to(torch.float64).cpu().numpy()
        assert np.abs(got - want).max() <= FIELD_TOL, (j, i, got, want)


def test_run_largest_grid_against_staged_path(P):
    """A run on the largest grid (32768^2): the fused, graph-replayed iteration (smoothing
    + tile reduce in one kernel, field written by the carry pass) against the staged
    drop-in path (build_density -> inim_field_from_density -> sample_field), whose field
    is itself checked at spot pixels against brute-force region sums; k = 16 raises
    MemoryError (the reference's float64 tables would need 256 GiB)."""
    import torch

    k = 15
    s = 1 << k
    pts = clusters(2_000_000, 15)
    params = P.RegularizationParams(k=k, kernel_size=8, iterations=1)
    r = P.run(P.ScatterDataset(positions=pts), params)
    new, field, dens = P.iterate_once(pts, params)
    assert maxerr(r.frame(1), new) <= 1e-6
    ft = r.fields[0].device_targets()
    assert float((ft - field.device_targets()).abs().max()) <= FIELD_TOL
    d = dens.device_values()
    brute = DeviceBrute(d)
    C = float(d.to(torch.float64).sum())
    for (j, i) in spot_pixels(s):
        x, y = i / s, j / s
        raw = raw_map_at(brute.tables_at(j, i), C, x, y)
        flat = raw_map_at(ones_tables_at(s, j, i), float(s) * s, x, y)
        want = np.clip(np.array([x, y]) + raw - flat, 0.0, 1.0)
        assert np.abs(ft[j, i].to(torch.float64).cpu().numpy() - want).max() <= FIELD_TOL, (j, i)
    del brute, d, ft, r, field, dens
    with pytest.raises(MemoryError):
        P.run(P.ScatterDataset(positions=pts[:10]), P.RegularizationParams(k=16, iterations=1))


# ------------------------------------------------------------------ kernel_size > 16
@pytest.mark.parametrize("ks", [17, 20, 32])
def test_density_generic_kernel_sizes(P, oracle, ks):
    pts = clusters(200_000, 3)
    tex = P.build_density(pts, P.RegularizationParams(k=9, kernel_size=ks))
    want, bg = oracle.build_density(pts, 9, ks)
    assert tex.background == bg
    assert maxerr(tex.values, want) <= 2e-6 * want.max()


@pytest.mark.parametrize("k,ks", [(4, 20), (3, 40), (6, 100)])
def test_smoothing_kernel_longer_than_reflection_period(P, oracle, rng, k, ks):
    """6 ks + 1 taps > 2 s: the taps fold onto one reflection period."""
    s = 1 << k
    g = f32(rng.random((s, s)) * 5)
    want = oracle.gaussian_smooth(g, ks)
    assert maxerr(P.gaussian_smooth(g, ks), want) <= 2e-6 * np.abs(want).max()


@pytest.mark.parametrize("ks", [20, 32])
def test_run_generic_kernel_size_against_oracle(P, oracle, ks):
    pts = clusters(100_000, 5)
    want = oracle_frames(oracle, pts, 9, ks, 3, {1, 2, 3})
    r = P.run(P.ScatterDataset(positions=pts), P.RegularizationParams(k=9, kernel_size=ks, iterations=3),
              store_fields=False)
    for t in (1, 2, 3):
        assert maxerr(r.frame(t), want[t]) <= POS_TOL, t


# -------------------------------------------------------------- run-mode regressions
def test_time_stop_records_fields(P):
    """stop="time" keeps one field per iteration (regularize.py:68-69), so map_through
    reproduces the last frame; an empty dataset records (0, 2) frames."""
    ds = P.ScatterDataset(positions=clusters(5000, 9))
    rt = P.run(ds, P.RegularizationParams(k=6, iterations=4, stop="time", time_budget=60.0))
    assert rt.iterations == 4 and len(rt.fields) == 4
    assert np.array_equal(P.map_through(rt, ds.positions), rt.frame(4))
    ref = P.run(ds, P.RegularizationParams(k=6, iterations=4))
    assert np.array_equal(rt.frame(4), ref.frame(4))
    empty = P.run(P.ScatterDataset(positions=np.empty((0, 2))),
                  P.RegularizationParams(k=5, iterations=2, stop="time", time_budget=60.0))
    assert empty.frame(2).shape == (0, 2) and len(empty.fields) == 2


def test_tiny_epsilon_still_stops_or_completes(P):
    """A positive epsilon below float32's smallest denormal must not disable the
    displacement criterion (or hang the run loop)."""
    ds = P.ScatterDataset(positions=clusters(5000, 2))
    r = P.run(ds, P.RegularizationParams(k=6, iterations=5, stop="displacement", epsilon=1e-300))
    assert r.iterations == 5
