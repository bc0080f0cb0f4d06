import functools
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

OPERATORS = os.path.join(ROOT, "operators")
GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200)")


@functools.lru_cache(maxsize=None)
def load_op(name: str):
    from paper_2605_28475_b200.operator import load_cache

    path = os.path.join(OPERATORS, f"{name}.bfct")
    if not os.path.exists(path):
        pytest.skip(f"operator {name} not available")
    return load_cache(path)


@functools.lru_cache(maxsize=None)
def golden(name: str):
    path = os.path.join(GOLDEN, f"{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden {name} not available")
    return dict(np.load(path))


def golden_names():
    return sorted(f[:-4] for f in os.listdir(GOLDEN)
                  if f.endswith(".npz") and not f.startswith("rk4_")
                  and f not in ("project.npz", "maxwell_rates.npz", "rtensor_quadconv.npz"))


def reference_available() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def reference():
    """The reference package, imported read-only (build container only)."""
    if not reference_available():
        pytest.skip("reference not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.append(REFERENCE_SRC)
    import boltzfact.cache
    import boltzfact.contraction

    return boltzfact
