"""The kernel-level drop-in (paper_2511_08427_b200.tomokit_kernels) binds into
the unmodified reference: every call site of the six numba kernels and of the
numpy row filter ends up on libtkb200.so.  CPU-only (binding, no launches);
the GPU run of the reference's own suites is scripts/run_reference_suite.py."""

import inspect
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


@pytest.fixture()
def tomokit():
    if not (REF / "tomokit").is_dir():
        pytest.skip("baseline/_ref not installed (scripts/install_reference.sh)")
    sys.path.insert(0, str(REF))
    import tomokit

    yield tomokit
    sys.path.remove(str(REF))


def test_signatures_match_the_reference_kernels(tomokit):
    from tomokit import _kernels

    from paper_2511_08427_b200 import tomokit_kernels as K

    for name in ("forward_parallel_2d", "back_parallel_2d", "forward_fan_2d", "back_fan_2d", "forward_cone_3d",
                 "back_cone_3d"):
        ref = inspect.signature(getattr(_kernels, name).py_func)
        assert list(inspect.signature(getattr(K, name)).parameters) == list(ref.parameters), name


def test_install_rebinds_every_call_site(tomokit):
    from tomokit import _kernels, autodiff, filters

    from paper_2511_08427_b200 import tomokit_kernels as K

    saved = K.install(tomokit)
    try:
        assert _kernels.forward_cone_3d is K.forward_cone_3d and _kernels.back_cone_3d is K.back_cone_3d
        assert filters.fft_filter is K.fft_filter and autodiff.fft_filter is K.fft_filter
        names = {f"{m.__name__}.{a}" for m, a, _ in saved}
        assert {"tomokit._kernels.forward_parallel_2d", "tomokit._kernels.back_fan_2d",
                "tomokit.filters.fft_filter", "tomokit.autodiff.fft_filter"} <= names
    finally:
        for mod, attr, val in saved:
            setattr(mod, attr, val)
    assert _kernels.forward_cone_3d is not K.forward_cone_3d
