"""The host staging transfers of the drop-in's float64 boundary (inim_h2d_narrow /
inim_d2h_widen, csrc/abi.cu): bit-identical to numpy's float64 <-> float32 casts (IEEE
round to nearest, like the device cast kernels) at every chunking edge, including
non-finite values and subnormals, and usable back to back on one stream."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 18  # floats per page-locked slot (csrc/abi.cu kStageChunk)


def _special(rng, n):
    x = rng.normal(0.0, 10.0, n)
    if n >= 8:
        x[:8] = [np.inf, -np.inf, np.nan, 0.0, -0.0, 1e-40, 3.4e38 * 1.5, 2.0 ** -149 / 3]
    return x


@pytest.mark.parametrize("n", [0, 1, 7, 1000, CHUNK - 1, CHUNK, CHUNK + 1, 3 * CHUNK + 12345])
def test_h2d_narrow_and_d2h_widen_bit_exact(rng, n):
    import torch

    from paper_2408_06513_b200 import _device as D, _lib

    lib = _lib.load()
    host = _special(rng, n)
    dev = torch.empty(max(n, 1), dtype=torch.float32, device="cuda")
    _lib.check(lib.inim_h2d_narrow(host.ctypes.data, D.ptr(dev), n, D.stream()), "h2d")
    got = dev[:n].cpu().numpy()
    with np.errstate(over="ignore"):
        want = host.astype(np.float32)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))

    back = np.full(n, 7.0)
    _lib.check(lib.inim_d2h_widen(D.ptr(dev), back.ctypes.data, n, D.stream()), "d2h")
    assert np.array_equal(back.view(np.uint64), want.astype(np.float64).view(np.uint64))


def test_back_to_back_transfers_keep_their_data(rng):
    """Consecutive narrows reuse the two slots: each DMA must have read its slot before
    the host overwrites it."""
    import torch

    from paper_2408_06513_b200 import _device as D, _lib

    lib = _lib.load()
    n = 5 * CHUNK + 3
    outs = []
    hosts = []
    for q in range(4):
        h = rng.random(n) + q
        hosts.append(h)
        d = torch.empty(n, dtype=torch.float32, device="cuda")
        _lib.check(lib.inim_h2d_narrow(h.ctypes.data, D.ptr(d), n, D.stream()), "h2d")
        outs.append(d)
    for h, d in zip(hosts, outs):
        assert np.array_equal(d.cpu().numpy(), h.astype(np.float32))


def test_argument_errors():
    from paper_2408_06513_b200 import _lib

    lib = _lib.load()
    assert lib.inim_h2d_narrow(None, None, 4, None) == _lib.INIM_EINVAL
    assert lib.inim_d2h_widen(None, None, -1, None) == _lib.INIM_EINVAL
    assert lib.inim_h2d_narrow(ctypes.c_void_p(None), ctypes.c_void_p(None), 0, None) == 0
