"""Pin the CPU oracle (oracle/inim_oracle.c) to golden vectors recorded from the
unmodified reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest


def rel(a, b, scale=1.0):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max()) / scale


def test_accumulate_bit_exact(oracle, golden):
    g = golden("accumulate")
    for k, key in ((6, "counts"), (3, "counts_k3"), (9, "counts_k9")):
        assert np.array_equal(oracle.accumulate(g["positions"], k), g[key])


def test_smoothing_kernel(oracle, golden):
    g = golden("smooth")
    for ks in (1, 2, 8):
        assert rel(oracle.smoothing_kernel(ks), g[f"w{ks}"]) < 1e-16


@pytest.mark.parametrize("grid,ks,key", [("g32", 2, "s32_ks2"), ("g32", 8, "s32_ks8"), ("g16", 8, "s16_ks8"),
                                          ("g8", 3, "s8_ks3")])
def test_gaussian_smooth(oracle, golden, grid, ks, key):
    g = golden("smooth")
    # identical algorithm; only exp() may differ by one ulp between libm and numpy
    assert rel(oracle.gaussian_smooth(g[grid], ks), g[key]) < 1e-14


def test_build_density(oracle, golden):
    g = golden("density")
    v, bg = oracle.build_density(g["positions"], 6, 4)
    assert bg == g["background_k6_ks4"]
    assert rel(v, g["values_k6_ks4"]) < 1e-13
    v, bg = oracle.build_density(g["positions"], 5, 2, 0.25)
    assert bg == 0.25
    assert rel(v, g["values_k5_ks2_bg"]) < 1e-13


@pytest.mark.parametrize("s", [2, 4, 8, 16, 32, 64, 128])
def test_integral_tables_bit_exact(oracle, golden, s):
    g = golden("integral")
    t, total = oracle.build_integral_set(g[f"d{s}"])
    assert np.array_equal(t, g[f"t{s}"])
    assert total == g[f"total{s}"]


def test_integral_integer_and_columns(oracle, golden):
    g = golden("integral")
    t, _ = oracle.build_integral_set(g["dint"])
    assert np.array_equal(t, g["tint"])
    up, lo = oracle.column_integrals(g["dint"])
    assert np.array_equal(up, g["upper_int"]) and np.array_equal(lo, g["lower_int"])
    t, total = oracle.build_integral_set(g["dconst"])
    assert np.array_equal(t, g["tconst"]) and total == g["totalconst"]


def test_flat_response_bit_exact(oracle, golden):
    g = golden("flat")
    for k in (1, 2, 3, 4, 5, 6, 8):
        assert np.array_equal(oracle.flat_response(k), g[f"defect_k{k}"])


def test_field_and_sample_bit_exact(oracle, golden):
    g = golden("field")
    t, exc = oracle.build_field(g["tables"], float(g["total"]), 6)
    assert np.array_equal(t, g["targets"]) and exc == g["max_excursion"]
    g = golden("sample")
    assert np.array_equal(oracle.sample_field(g["targets"], g["points"]), g["out"])
    assert np.array_equal(oracle.sample_field(g["field_targets"], g["field_points"]), g["field_out"])


def test_iterate_and_runs(oracle, golden):
    g = golden("iterate")
    new, f, dd = oracle.iterate_once(g["positions"], 6, 4, want_field=True, want_density=True)
    assert rel(new, g["new_positions"]) < 1e-14
    assert rel(f, g["targets"]) < 1e-14
    assert rel(dd, g["density"]) < 1e-13
    g = golden("run_c1")
    frames = oracle.run_positions(g["positions"], 8, 8, 5)
    assert rel(np.stack(frames), g["frames"]) < 1e-13
    g = golden("run_disp")
    frames = oracle.run_positions(g["positions"], 6, 8, 50, stop="displacement", epsilon=5e-3)
    assert len(frames) - 1 == int(g["n_iters"])
    assert rel(frames[-1], g["last"]) < 1e-13


def test_oracle_known_answers(oracle):
    # test_integral.py:24-39, 88-97, 133-143 restated on the oracle
    up, lo = oracle.column_integrals(np.ones((4, 4)))
    for j in range(4):
        assert np.all(up[j] == j + 1) and np.all(lo[j] == 3 - j)
    t, _ = oracle.build_integral_set(np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert t[0, 1, 1] == 10 and t[0, 0, 0] == 1 and t[1, 0, 0] == 3 and t[3, 0, 0] == 2 and t[2, 0, 0] == 4
    t, _ = oracle.build_integral_set(np.ones((4, 4)))
    assert t[4, 1, 1] == 4.0


def test_brute_force_regions(oracle, rng):
    """Oracle tables against the O(s^4) region definitions (tests/oracles.py:12-40)."""
    for s in (4, 8, 16):
        d = rng.random((s, s))
        t, total = oracle.build_integral_set(d)
        want = np.zeros((8, s, s))
        jj, ii = np.mgrid[0:s, 0:s]
        for j in range(s):
            for i in range(s):
                a, b = ii <= i, jj <= j
                u, w = ii + jj <= i + j, ii - jj >= i - j
                masks = (a & b, a & ~b, ~a & ~b, ~a & b, u & w, u & ~w, ~u & ~w, ~u & w)
                for q, msk in enumerate(masks):
                    want[q, j, i] = d[msk].sum()
        assert rel(t, want, total) < 1e-12
