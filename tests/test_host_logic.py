"""CPU tests of the host-side logic: the C ABI library loads and exports every symbol
include/inim.h declares, the carry algebra of the device integral pipeline (numpy
model, tests/tile_model.py) against the oracle, the closed-form flat response used by
the fused field kernel, parameter validation and the frame thinning policy."""

import ctypes
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    from paper_2408_06513_b200 import _lib

    _lib.build()
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.inim_version().startswith(b"libinim sm_100a")
    out = subprocess.run(["nm", "-D", str(_lib.LIB_PATH)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(declared) <= exported


def test_library_is_sm100a_only():
    from paper_2408_06513_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    archs = {ln.split(".")[-2] for ln in out.splitlines() if ".cubin" in ln}
    assert archs == {"sm_100a"}, archs


def test_chain_scan_keeps_three_ctas_per_sm():
    """The standalone chain scan is occupancy-sensitive (72 registers =
    1 CTA/SM cost 4% of the whole 16384^2 integral pass); 512 threads x <= 40 registers
    keeps 3 CTAs/SM."""
    from paper_2408_06513_b200 import _lib

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-res-usage", str(_lib.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout.splitlines()
    regs = [int(nxt.split("REG:")[1].split()[0]) for ln, nxt in zip(out, out[1:])
            if "chains_kernelILb0E" in ln and "REG:" in nxt]  # the single-plot instantiation
    assert regs and max(regs) <= 40, regs


def test_workspace_and_argument_errors_without_gpu():
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    assert lib.inim_workspace_bytes(10, 1_000_000, 1) > 8 * 1024 * 1024
    assert lib.inim_workspace_bytes(99, 0, 1) == 0
    # argument validation happens before any device work
    assert lib.inim_splat(None, 0, 10, 4, None, None) == _lib.INIM_EINVAL
    assert lib.inim_integral_set(None, 4, None, None, None, None) == _lib.INIM_EINVAL
    assert lib.inim_run(None, 10, 0, 8, 0.0, 1, 0.0, None, None, None, None, None, None, None) == _lib.INIM_EINVAL
    assert lib.inim_kernels_per_iteration(10) > 5


@pytest.mark.parametrize("s,th,tw", [(1, None, None), (2, None, None), (8, None, None), (32, None, None),
                                     (64, None, None), (64, 16, 32), (128, None, None), (256, None, None),
                                     (128, 32, 32)])
def test_tile_carry_algebra_matches_oracle(oracle, rng, s, th, tw):
    from tile_model import model_tables

    d = rng.random((s, s)) * rng.uniform(0.5, 20)
    got, C = model_tables(d, th, tw)
    want, total = oracle.build_integral_set(d)
    assert abs(C - total) <= 1e-12 * total
    assert np.abs(got - want).max() <= 1e-12 * total


def closed_form_flat(k):
    """numpy restatement of the device closed form (csrc/integral.cu flat_response_at)."""
    S = 1 << k
    jj, ii = np.mgrid[0:S, 0:S].astype(np.int64)
    s2 = S * S
    tl = (ii + 1) * (jj + 1)
    bl = (ii + 1) * (S - 1 - jj)
    tr = (S - 1 - ii) * (jj + 1)
    br = (S - 1 - ii) * (S - 1 - jj)

    def f(L):
        return L * (jj + 1) - L * (L + 1) // 2

    up = (jj + 1) + f(np.minimum(jj, ii)) + f(np.minimum(jj, S - 1 - ii))
    sg = ii + jj
    A1 = np.where(sg <= S - 1, (sg + 1) * (sg + 2) // 2, s2 - (2 * S - 2 - sg) * (2 * S - 1 - sg) // 2)
    dl = ii - jj
    D1 = np.where(dl >= 0, (S - dl) * (S - dl + 1) // 2, s2 - (S + dl - 1) * (S + dl) // 2)
    left, right = A1 - up, D1 - up
    down = s2 - up - left - right
    return np.stack([tl, bl, br, tr, up, left, down, right]).astype(np.float64), float(s2)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 8])
def test_closed_form_region_counts(oracle, golden, k):
    t8, total = closed_form_flat(k)
    want, wtot = oracle.build_integral_set(np.ones((1 << k, 1 << k)))
    assert np.array_equal(t8, want) and total == wtot
    defect = oracle.raw_targets_per_pixel(t8, total, k)
    assert np.array_equal(defect, golden("flat")[f"defect_k{k}"])


def test_params_validation():
    from paper_2408_06513_b200 import InvalidParams, RegularizationParams

    RegularizationParams().validate()
    bad = [dict(k=0), dict(kernel_size=0), dict(iterations=-1), dict(stop="never"),
           dict(stop="displacement", epsilon=0.0), dict(stop="time"), dict(background=0.0), dict(frame_cap=1)]
    for kw in bad:
        with pytest.raises(InvalidParams):
            RegularizationParams(**kw).validate()


def _reference_thinning(iterations, cap):
    frames, stride, top = {0}, 1, 0
    for t in range(1, iterations + 1):
        frames.add(t)
        top = t
        if len(frames) > cap:
            stride *= 2
            frames = {i for i in frames if i in (0, top) or i % stride == 0}
    return frames


@pytest.mark.parametrize("T,cap", [(5, 64), (9, 4), (10, 2), (33, 8), (100, 64), (7, 3)])
def test_survivor_policy_matches_reference(T, cap):
    from paper_2408_06513_b200.regularize import _survivors

    assert _survivors(T, cap) == _reference_thinning(T, cap)


def test_validate_dataset_and_errors():
    from paper_2408_06513_b200 import (CoordinateOutOfRange, NonFiniteCoordinate, ScatterDataset, UncrowdError,
                                       validate_dataset)

    ds = validate_dataset([[0, 0], [2, 4], [1, 1]])
    assert np.allclose(ds.positions, [[0, 0], [1, 1], [0.5, 0.25]])
    assert isinstance(ds, ScatterDataset) and list(ds.ids) == [0, 1, 2]
    with pytest.raises(NonFiniteCoordinate):
        validate_dataset([[0, np.nan]])
    with pytest.raises(CoordinateOutOfRange):
        validate_dataset([[0, 2.0]], normalize=False)
    assert issubclass(NonFiniteCoordinate, UncrowdError) and issubclass(NonFiniteCoordinate, ValueError)


def test_compute_without_gpu_raises_not_falls_back():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import paper_2408_06513_b200 as P

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.accumulate(np.zeros((3, 2)), 4)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.build_integral_set(np.ones((8, 8)))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.binned_stddev(np.full((3, 2), 0.5), 4)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.trustworthiness(np.random.rand(20, 2), np.random.rand(20, 2))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        P.run(P.ScatterDataset(positions=np.full((3, 2), 0.5)), P.RegularizationParams(k=4, iterations=1),
              collect_metrics="full")


def test_oracle_not_imported_by_product():
    for path in (ROOT / "paper_2408_06513_b200").rglob("*.py"):
        text = path.read_text()
        assert "oracle" not in text.replace("oracles.py", "").lower() or "no oracle" in text.lower(), path


def test_generated_taps_match_oracle_kernel(oracle):
    """csrc/inim_taps.cuh (FFMA-immediate taps) is current and equals the oracle's
    smoothing_kernel rounded to float32 (density.py:30-37)."""
    import sys
    sys.path.insert(0, str(ROOT / "tools"))
    import gen_taps
    assert gen_taps.OUT.read_text() == gen_taps.render(), "run tools/gen_taps.py"
    for ks in (1, 2, 5, 8, 16):
        ref = np.asarray(oracle.smoothing_kernel(ks), dtype=np.float64).astype(np.float32)
        np.testing.assert_array_equal(gen_taps.taps(ks), ref)
