"""Record golden vectors from the UNMODIFIED reference package (run in the build
container, where /root/reference exists; the GPU box only reads the committed .npz).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py [metrics|encodings]

The reference `uncrowd` package imports skimage at encodings.py:16, which is absent
here, so a stub module is installed first; nothing on the
hot path touches it.  All input coordinates are float32-representable so that the
B200 path (fp32 positions) and the reference see identical inputs.

Output: tests/golden/golden_<case>.npz, one file per case.
"""

from __future__ import annotations

import os
import sys
import types
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def import_reference():
    sk = types.ModuleType("skimage")
    me = types.ModuleType("skimage.measure")

    def find_contours(*a, **k):  # pragma: no cover - never called on the hot path
        raise NotImplementedError("skimage stub")

    me.find_contours = find_contours
    sk.measure = me
    sys.modules.setdefault("skimage", sk)
    sys.modules.setdefault("skimage.measure", me)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    import uncrowd  # noqa: E402

    return uncrowd


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def tables_of(t):
    return np.stack(t.tables())


def save(name, **arrays):
    np.savez_compressed(OUT / f"golden_{name}.npz", **arrays)
    print(f"golden_{name}.npz", {k: np.asarray(v).shape for k, v in arrays.items()})


def three_cluster(n, seed):
    """Three Gaussian clusters inside the unit square, fp32-representable."""
    rng = np.random.default_rng(seed)
    centers = np.array([[0.3, 0.35], [0.7, 0.4], [0.5, 0.72]])
    sig = np.array([0.05, 0.03, 0.08])
    counts = np.array([n // 2, n // 3, n - n // 2 - n // 3])
    pts = np.concatenate([rng.normal(centers[c], sig[c], size=(counts[c], 2)) for c in range(3)])
    return f32(np.clip(pts, 0.0, 1.0))


def main():
    uc = import_reference()
    from uncrowd.density import accumulate, gaussian_smooth, smoothing_kernel
    from uncrowd.integral import build_integral_set, column_integrals
    from uncrowd.mapping import build_field, flat_response, sample_field

    rng = np.random.default_rng(2408)

    # --- accumulate: random points plus edge/boundary coordinates (density.py:14-27)
    pts = f32(rng.random((5000, 2)))
    edges = np.array([[0, 0], [1, 1], [1, 0], [0, 1], [0.5, 0.5], [0.999999, 0.25],
                      [2 ** -6, 3 * 2 ** -6], [1 - 2 ** -7, 1 - 2 ** -7]], dtype=np.float64)
    pts = np.concatenate([pts, f32(edges)])
    save("accumulate", positions=pts, k=6, counts=accumulate(pts, 6),
         counts_k3=accumulate(pts, 3), counts_k9=accumulate(pts, 9))

    # --- smoothing (density.py:30-51), including radius > side (repeated reflection)
    g32 = f32(rng.random((32, 32)))
    g16 = f32(rng.random((16, 16)) ** 3)
    g8 = f32(rng.integers(0, 9, size=(8, 8)))
    save("smooth", w1=smoothing_kernel(1), w2=smoothing_kernel(2), w8=smoothing_kernel(8),
         g32=g32, s32_ks2=gaussian_smooth(g32, 2), s32_ks8=gaussian_smooth(g32, 8),
         g16=g16, s16_ks8=gaussian_smooth(g16, 8), g8=g8, s8_ks3=gaussian_smooth(g8, 3))

    # --- build_density on a blob (conftest.py:15-21 pattern)
    gen = np.random.default_rng(11)
    blob = f32(np.clip(gen.normal(loc=(0.35, 0.5), scale=0.04, size=(2000, 2)), 0.0, 1.0))
    tex = uc.build_density(blob, uc.RegularizationParams(k=6, kernel_size=4))
    tex_b = uc.build_density(blob, uc.RegularizationParams(k=5, kernel_size=2, background=0.25))
    save("density", positions=blob, values_k6_ks4=tex.values, background_k6_ks4=tex.background,
         values_k5_ks2_bg=tex_b.values, background_k5_ks2_bg=tex_b.background)

    # --- integral tables (integral.py:180-247), s = 2..128, random, integer, constant
    integ = {}
    for s in (2, 4, 8, 16, 32, 64, 128):
        d = f32(rng.random((s, s)) * rng.uniform(0.5, 20))
        t = build_integral_set(d)
        integ[f"d{s}"] = d
        integ[f"t{s}"] = tables_of(t)
        integ[f"total{s}"] = t.total
    di = f32(rng.integers(0, 100, size=(32, 32)))
    ti = build_integral_set(di)
    cols = column_integrals(di)
    integ.update(dint=di, tint=tables_of(ti), totalint=ti.total, upper_int=cols.upper, lower_int=cols.lower)
    dc = np.full((16, 16), 1.3)
    tc = build_integral_set(dc)
    integ.update(dconst=dc, tconst=tables_of(tc), totalconst=tc.total)
    save("integral", **integ)

    # --- flat response / defect (mapping.py:104-129)
    flat_response.clear()
    save("flat", **{f"defect_k{k}": flat_response.get(k) for k in (1, 2, 3, 4, 5, 6, 8)})

    # --- build_field on the blob density (mapping.py:194-204)
    t6 = build_integral_set(tex)
    field = build_field(t6)
    save("field", tables=tables_of(t6), total=t6.total, k=6, targets=field.targets,
         max_excursion=field.max_excursion)

    # --- sample_field (mapping.py:207-246): random field, interior + edge points
    tgt = f32(rng.random((16, 16, 2)))
    sp = np.concatenate([f32(rng.random((500, 2))), f32(edges)])
    save("sample", targets=tgt, points=sp, out=sample_field(uc.DeformationField(targets=tgt, k=4), sp),
         field_targets=field.targets, field_points=blob,
         field_out=sample_field(field, blob))

    # --- iterate_once (regularize.py:25-37)
    params = uc.RegularizationParams(k=6, kernel_size=4)
    new, fld, dens = uc.iterate_once(blob, params)
    save("iterate", positions=blob, k=6, kernel_size=4, new_positions=new,
         targets=fld.targets, max_excursion=fld.max_excursion, density=dens.values)

    # --- C1-like run: 3-cluster 10k points, 256^2, ks=8, 5 iterations (BASELINE configs[0])
    p10k = three_cluster(10_000, 2408)
    run = uc.run(uc.ScatterDataset(positions=p10k), uc.RegularizationParams(k=8, kernel_size=8, iterations=5))
    save("run_c1", positions=p10k, k=8, kernel_size=8, iterations=5,
         frames=np.stack([run.frame(t) for t in range(run.iterations + 1)]),
         field_last=run.fields[-1].targets,
         excursions=np.array([f.max_excursion for f in run.fields]))

    # --- displacement stop on the blob (test_regularize.py:63-69 pattern)
    pr = uc.RegularizationParams(k=6, iterations=50, stop="displacement", epsilon=5e-3)
    rd = uc.run(uc.ScatterDataset(positions=blob), pr)
    save("run_disp", positions=blob, k=6, kernel_size=8, iterations=50, epsilon=5e-3,
         n_iters=rd.iterations, last=rd.frame(rd.iterations))


def metrics_cases():
    """Layout metrics (metrics.py:46-168), including run(collect_metrics="full")."""
    uc = import_reference()
    from uncrowd import metrics as M

    rng = np.random.default_rng(1789)
    occ = {}
    for k in (2, 4, 6, 8):
        pts = np.concatenate([f32(rng.random((3000, 2))), three_cluster(2000, k),
                              f32(np.array([[0, 0], [1, 1], [1, 0], [0, 1], [0.5, 0.5]] * 3))])
        occ[f"pts_k{k}"] = pts
        occ[f"binned_k{k}"] = M.binned_stddev(pts, k)
        occ[f"over_k{k}"] = M.overplotting(pts, k)
    grid = f32((np.stack(np.meshgrid(np.arange(16), np.arange(16)), -1).reshape(-1, 2) + 0.5) / 16)
    occ.update(uniform=grid, binned_uniform=M.binned_stddev(grid, 4), over_uniform=M.overplotting(grid, 4))

    # neighbourhood metrics: a perturbed layout with ties (duplicated points), n < cap
    base = f32(rng.random((600, 2)))
    base[100:110] = base[0]
    moved = f32(np.clip(base + rng.normal(0, 0.02, base.shape), 0, 1))
    nb = dict(orig=base, moved=moved,
              trust10=M.trustworthiness(base, moved, 10), trust3=M.trustworthiness(base, moved, 3),
              order=M.orthogonal_ordering(base, moved), trust_self=M.trustworthiness(base, base, 10),
              order_self=M.orthogonal_ordering(base, base))
    # subsampled ordering (n > cap)
    big = f32(rng.random((6000, 2)))
    bigm = f32(np.clip(big + rng.normal(0, 0.05, big.shape), 0, 1))
    nb.update(big=big, bigm=bigm, order_big=M.orthogonal_ordering(big, bigm),
              order_big_cap=M.orthogonal_ordering(big, bigm, sample_cap=1000))

    # run with full metrics on the C1 layout (10k points > the 4096 subsample cap)
    p10k = three_cluster(10_000, 2408)
    run = uc.run(uc.ScatterDataset(positions=p10k), uc.RegularizationParams(k=8, kernel_size=8, iterations=3),
                 collect_metrics="full")
    recs = run.metrics
    save("metrics", **{f"occ_{k}": v for k, v in occ.items()}, **{f"nb_{k}": v for k, v in nb.items()},
         run_positions=p10k, run_k=8, run_iterations=3,
         run_frames=np.stack([run.frame(t) for t in range(run.iterations + 1)]),
         run_binned=np.array([r.binned_stddev for r in recs]), run_over=np.array([r.overplotting for r in recs]),
         run_trust=np.array([r.trustworthiness for r in recs]), run_order=np.array([r.ordering for r in recs]),
         run_json=np.array([r.to_json_line() for r in recs]))


def encodings_cases():
    """deform_grid / deform_background / field dumps (encodings.py:55-162,
    fileio.py:63-104, service.py:170-172) on the reference test suite's blob run
    (test_encodings.py:32-37), with the intermediates the oracle is pinned on."""
    uc = import_reference()
    import io
    import tempfile

    from uncrowd import encodings as E, fileio
    from uncrowd.density import build_density

    gen = np.random.default_rng(11)
    pts = f32(np.clip(gen.normal((0.35, 0.5), 0.04, (2000, 2)), 0.0, 1.0))
    ds = uc.validate_dataset(pts, normalize=False)
    run = uc.run(ds, uc.RegularizationParams(k=7, kernel_size=8, iterations=4))
    k = 7
    X, Y = uc.model.unit_coordinates(k)
    sources = np.column_stack([X.ravel(), Y.ravel()])
    targets = uc.map_through(run.fields, sources)
    dens = build_density(run.frame(0), run.params)
    bg = E.deform_background(run)
    bg2 = E.deform_background(run, upto=2)
    grid = E.deform_grid(run, spacing=16, subdivision=4)
    with tempfile.TemporaryDirectory() as tmp:
        fileio.export_field(run.fields[-1], f"{tmp}/f.bin", iteration=4)
        field_bytes = open(f"{tmp}/f.bin", "rb").read()
        fileio.export_grid(dens.values, f"{tmp}/g.bin", k=k, index=3)
        grid_bytes = open(f"{tmp}/g.bin", "rb").read()
    payload = {f"payload_{str(lv).replace('.', '_')}": np.frombuffer(
        uc.transition_positions(run, lv).astype("<f4").tobytes(), dtype=np.uint8) for lv in (0, 1.25, 2.5, 4)}
    save("encodings", positions=pts, k=k, iterations=4,
         frames=np.stack([run.frame(t) for t in range(run.iterations + 1)]),
         fields=np.stack([f.targets for f in run.fields]),
         targets=targets, density=dens.values, background=bg.values, background_range=np.array(bg.value_range),
         background_upto2=bg2.values,
         grid_sizes=np.array([len(line) for line in grid.polylines]), grid=np.concatenate(grid.polylines),
         field_bytes=np.frombuffer(field_bytes, dtype=np.uint8), grid_bytes=np.frombuffer(grid_bytes, dtype=np.uint8),
         **payload)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "metrics":
        metrics_cases()
    elif len(sys.argv) > 1 and sys.argv[1] == "encodings":
        encodings_cases()
    else:
        main()
        metrics_cases()
        encodings_cases()
