import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture
def rng():
    return np.random.default_rng(20240)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(GOLDEN / f"golden_{name}.npz"))
        return cache[name]

    return load


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def P():
    """The product package, only for GPU tests: fails loudly without CUDA."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    import paper_2408_06513_b200 as pkg
    from paper_2408_06513_b200 import _lib

    _lib.load()
    return pkg


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def blob(n=2000, seed=11, loc=(0.35, 0.5), scale=0.04):
    gen = np.random.default_rng(seed)
    return f32(np.clip(gen.normal(loc=loc, scale=scale, size=(n, 2)), 0.0, 1.0))


def clusters(n, seed, centers=((0.3, 0.3), (0.7, 0.3), (0.3, 0.7), (0.7, 0.7)), sigma=0.05):
    gen = np.random.default_rng(seed)
    parts = np.array_split(np.arange(n), len(centers))
    pts = np.concatenate([gen.normal(c, sigma, size=(len(p), 2)) for c, p in zip(centers, parts)])
    return f32(np.clip(pts, 0.0, 1.0))
