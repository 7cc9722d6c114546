"""GPU parity of the encodings and the binary dumps (encodings.py:55-162,
fileio.py:63-104, service.py:170-172) through the drop-in API and the C ABI
(inim_deform_background, inim_blend_frames).

Bars:
  deform_background  covered pixels bit-identical to the oracle's np.add.at-order splat
                     on the SAME inputs (our mapped source pixels and our density);
                     uncovered pixels hold the value of a covered pixel at exactly the
                     scipy distance-transform distance; against the reference's own
                     result within what the float32 pipeline allows (see below)
  grid / contours    vertices within the 2e-5 position tolerance of the reference; a
                     vertex on a sample lands exactly on that sample's frame
  field dump         byte-identical header; payload = the device field's own bytes
  positions payload  bit-identical to transition_positions(...).astype('<f4')
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

POS_TOL = 2e-5


@pytest.fixture(scope="module")
def blob_run(P, golden):
    g = golden("encodings")
    ds = P.ScatterDataset(positions=g["positions"])
    return P.run(ds, P.RegularizationParams(k=int(g["k"]), kernel_size=8, iterations=int(g["iterations"])))


def _own_inputs(P, run, upto=None):
    from paper_2408_06513_b200 import encodings as E
    from paper_2408_06513_b200._device import to_host64

    targets = to_host64(E.background_sources(run, upto))
    dens = P.build_density(run.frame(0), run.params)
    return targets, dens.values


def _check_against_oracle(oracle, got, targets, values, k):
    want, cov = oracle.background_splat(targets, values, k)
    assert np.array_equal(got[cov], want[cov])
    filled, dist = oracle.background_fill(want, cov)
    unc = np.argwhere(~cov)
    for j, i in unc:  # any covered pixel at the nearest distance is a valid source
        d2 = int(round(dist[j, i] ** 2))
        r = int(np.ceil(dist[j, i]))
        ys, xs = np.mgrid[max(0, j - r):j + r + 1, max(0, i - r):i + r + 1]
        ys, xs = ys.ravel(), xs.ravel()
        ok = (ys < cov.shape[0]) & (xs < cov.shape[1])
        ys, xs = ys[ok], xs[ok]
        near = cov[ys, xs] & ((ys - j) ** 2 + (xs - i) ** 2 == d2)
        assert near.any()
        assert got[j, i] in set(want[ys[near], xs[near]].tolist())
    return len(unc)


def test_background_matches_oracle_on_own_inputs(P, oracle, blob_run):
    k = blob_run.params.k
    tex = P.deform_background(blob_run)
    targets, values = _own_inputs(P, blob_run)
    _check_against_oracle(oracle, tex.values, targets, values, k)
    lo, hi = tex.value_range
    assert (lo, hi) == (float(values.min()), float(values.max()))
    assert tex.values.min() >= lo - 1e-12 and tex.values.max() <= hi + 1e-12


def test_background_upto_and_larger_grid(P, oracle, blob_run):
    tex = P.deform_background(blob_run, upto=2)
    targets, values = _own_inputs(P, blob_run, upto=2)
    _check_against_oracle(oracle, tex.values, targets, values, blob_run.params.k)
    from conftest import clusters

    run = P.run(P.ScatterDataset(positions=clusters(200_000, 3)),
                P.RegularizationParams(k=9, kernel_size=8, iterations=5), store_fields=True)
    tex = P.deform_background(run)
    targets, values = _own_inputs(P, run)
    _check_against_oracle(oracle, tex.values, targets, values, 9)


def test_background_against_reference(P, golden, blob_run):
    """Same inputs up to the float32 pipeline: density (fp32) and mapped positions
    (<= 2e-5).  The splat weights move by <= 2e-5 * s, so the texture follows the
    reference to a small fraction of its value range."""
    g = golden("encodings")
    tex = P.deform_background(blob_run)
    lo, hi = g["background_range"]
    err = np.abs(tex.values - g["background"]) / (hi - lo)
    assert np.quantile(err, 0.99) < 1e-3 and err.max() < 2e-2
    assert tex.value_range == pytest.approx(tuple(g["background_range"]), rel=1e-6)


def test_background_identity_run(P, blob_run):
    zero = P.run(blob_run.original, P.RegularizationParams(k=7, kernel_size=8, iterations=0))
    tex = P.deform_background(zero)
    want = P.build_density(blob_run.original.positions, zero.params)
    assert np.abs(tex.values - want.values).max() < 1e-6
    assert tex.values.sum() == pytest.approx(want.values.sum(), rel=1e-9)


def test_grid_and_contours(P, golden, blob_run):
    g = golden("encodings")
    grid = P.deform_grid(blob_run, spacing=16, subdivision=4)
    assert [len(line) for line in grid.polylines] == g["grid_sizes"].tolist()
    assert np.abs(np.concatenate(grid.polylines) - g["grid"]).max() <= POS_TOL
    # a vertex on a sample lands exactly on the sample's frame
    sample = blob_run.original.positions[123]
    assert np.array_equal(P.map_through(blob_run, sample[None, :])[0], blob_run.frame(blob_run.iterations)[123])
    # contours: any polylines, mapped as one batch == one by one
    lines = np.split(g["grid"], np.cumsum(g["grid_sizes"])[:-1])
    cs = P.ContourSet(polylines=lines[:5], line_levels=[1.0] * 5, levels=[1.0])
    moved = P.deform_contours(cs, blob_run)
    for a, b in zip(moved.polylines, lines[:5]):
        assert np.array_equal(a, P.map_through(blob_run, b))
    with pytest.raises(ValueError):
        P.deform_grid(blob_run, spacing=1)


def test_field_dump_round_trip(P, golden, blob_run, tmp_path):
    from paper_2408_06513_b200 import fileio

    f = blob_run.fields[-1]
    path = tmp_path / "f.bin"
    fileio.export_field(f, path, iteration=4)
    blob = path.read_bytes()
    g = golden("encodings")
    assert blob[:16] == g["field_bytes"].tobytes()[:16]
    assert blob[16:] == f.targets.astype("<f4").tobytes()
    again, it = fileio.read_field(path)
    assert it == 4 and np.array_equal(again.targets, f.targets)
    pts = blob_run.original.positions
    assert np.array_equal(P.map_through([again], pts), P.map_through([f], pts))
    # the reference's own dump, read and applied on the device
    ref = tmp_path / "r.bin"
    ref.write_bytes(g["field_bytes"].tobytes())
    rf, _ = fileio.read_field(ref)
    assert np.array_equal(rf.targets, g["fields"][-1].astype(np.float32).astype(np.float64))
    gp = tmp_path / "g.bin"
    dens = P.build_density(pts, blob_run.params)
    fileio.export_grid(dens.device_values(), gp, k=7, index=3)
    vals, idx = fileio.read_grid(gp)
    assert idx == 3 and np.array_equal(vals, dens.values)


@pytest.mark.parametrize("level", [0, 1.25, 2.5, 4])
def test_positions_payload(P, golden, blob_run, level):
    from paper_2408_06513_b200 import fileio

    got = fileio.positions_payload(blob_run, level)
    assert got == P.transition_positions(blob_run, level).astype("<f4").tobytes()
    ref = np.frombuffer(golden("encodings")[f"payload_{str(level).replace('.', '_')}"].tobytes(), dtype="<f4")
    assert np.abs(np.frombuffer(got, dtype="<f4") - ref).max() <= POS_TOL
