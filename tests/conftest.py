import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

try:  # hypothesis is optional; mirror the reference's deterministic profile
    from hypothesis import settings

    settings.register_profile("deterministic", derandomize=True, deadline=None)
    settings.load_profile("deterministic")
except ImportError:  # pragma: no cover
    pass


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running full-size case")


@pytest.fixture(autouse=True)
def _seed_torch():
    # unseeded torch draws in a test are then the same whatever ran before it
    try:
        import torch

        torch.manual_seed(0)
    except ImportError:  # pragma: no cover
        pass


@pytest.fixture()
def rng():
    # the reference suite's seed (pkg/tests/conftest.py:18-20)
    return np.random.default_rng(20240917)


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            with np.load(GOLDEN / f"{name}.npz") as z:
                cache[name] = {k: z[k] for k in z.files}
        return cache[name]

    return load


@pytest.fixture(scope="session")
def oracle():
    import oracle as ora

    ora.lib()
    return ora


def has_cuda() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_cuda():
        pytest.skip("no CUDA device")
    import torch

    return torch.device("cuda", 0)


os.environ.setdefault("OMP_NUM_THREADS", str(max(1, os.cpu_count() or 1)))
