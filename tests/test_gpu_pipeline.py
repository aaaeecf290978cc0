"""GPU tests of the upload-ordered forward projection (ops._fp_cone_overlapped):
the per-band z extents (tk_fp_band_z), cells built from a partial volume
(tk_fp_plan_cells), row-band launches (tk_fp_plan_project_rows) and strided
row copies (tk_copy_2d).  Every result is compared bit for bit with the
one-launch projection of the whole volume (same kernel, same arithmetic)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tk(cuda):
    import paper_2511_08427_b200 as tk

    return tk


def _geoms(tk):
    shape, sp = (72, 60, 66), (0.9, 1.0, 1.1)
    circ = tk.circular_cone_geometry(shape, sp, (96, 104), (1.5, 1.4), 37, 2 * np.pi, 1200.0, 750.0)
    hel = tk.helical_trajectory_3d(29, 4 * np.pi, 1200.0, 750.0, (96, 104), (1.5, 1.4), -10.0, 10.0)
    return [circ, tk.GeometryCone3D(shape, sp, (96, 104), (1.5, 1.4), hel, 1200.0, 750.0)]


@pytest.mark.parametrize("which", [0, 1], ids=["circular", "helical"])
def test_band_z_extent_is_conservative(tk, which):
    """Volume rows outside a band's extent poisoned with NaN: the band's projection is
    unchanged (every cell its samples read holds only rows inside the extent)."""
    from paper_2511_08427_b200.projectors import FP_BAND_ROWS, band_z_extent, fp_tensor

    geom = _geoms(tk)[which]
    step = 0.45
    x = torch.rand(geom.volume_shape, device="cuda")
    full = fp_tensor(x, geom, step)
    bz = band_z_extent(geom, step)
    rows = geom.detector_shape[0]
    assert len(bz) == -(-rows // FP_BAND_ROWS)
    nz = geom.volume_shape[0]
    checked = 0
    for b in range(0, len(bz), 3):
        lo, hi = int(bz[b, 0]), int(bz[b, 1])
        r0, r1 = b * FP_BAND_ROWS, min(rows, (b + 1) * FP_BAND_ROWS)
        if lo > hi:
            assert float(full[:, r0:r1].abs().max()) == 0.0
            continue
        assert 0 <= lo <= hi < nz
        y = x.clone()
        y[:lo] = float("nan")
        y[hi + 1:] = float("nan")
        got = fp_tensor(y, geom, step)
        assert torch.equal(got[:, r0:r1], full[:, r0:r1]), b
        checked += 1
    assert checked > 0


def test_partial_cells_and_row_launches(tk):
    """Only the central volume rows present (the rest NaN): cells built from them and the
    bands whose extent lies inside projected by row launches equal the full projection."""
    from paper_2511_08427_b200.projectors import FP_BAND_ROWS, ForwardProjectionPlan, band_z_extent, fp_tensor

    geom = _geoms(tk)[0]
    step = 0.45
    nz = geom.volume_shape[0]
    rows = geom.detector_shape[0]
    x = torch.rand(geom.volume_shape, device="cuda")
    full = fp_tensor(x, geom, step)
    a0, b0 = nz // 4, nz - nz // 4
    bz = band_z_extent(geom, step)
    ready = [b for b in range(len(bz)) if bz[b, 0] > bz[b, 1] or (bz[b, 0] >= a0 and bz[b, 1] < b0)]
    assert ready
    part = torch.full_like(x, float("nan"))
    part[a0:b0] = x[a0:b0]
    out = torch.full(geom.sinogram_shape, float("nan"), device="cuda")
    with ForwardProjectionPlan(part, geom) as plan:
        plan.cells(a0, b0)
        for b in ready:
            plan.project_rows(b * FP_BAND_ROWS, min(rows, (b + 1) * FP_BAND_ROWS), out, step)
        # the rest of the volume arrives: grow the cells, then every remaining band
        part[:a0] = x[:a0]
        part[b0:] = x[b0:]
        plan.cells(0, nz)
        for b in range(len(bz)):
            if b not in ready:
                plan.project_rows(b * FP_BAND_ROWS, min(rows, (b + 1) * FP_BAND_ROWS), out, step)
    assert torch.equal(out, full)


def test_row_launch_arguments(tk):
    from paper_2511_08427_b200.projectors import ForwardProjectionPlan

    geom = _geoms(tk)[0]
    x = torch.rand(geom.volume_shape, device="cuda")
    out = torch.empty(geom.sinogram_shape, device="cuda")
    with ForwardProjectionPlan(x, geom) as plan:
        with pytest.raises(ValueError, match="8-row bands"):
            plan.project_rows(3, 16, out, 0.45)
        with pytest.raises(ValueError, match="z0 < z1"):
            plan.cells(10, 10)
        plan.cells(30, 40)
        with pytest.raises(ValueError, match="one interval"):
            plan.cells(0, 5)


@pytest.mark.parametrize("which", [0, 1], ids=["45views", "44views"])
def test_py_forward_project_pipeline_bit_identical(tk, which, monkeypatch):
    """The pinned-host boundary call (upload-ordered row-band pipeline, or its view-chunk
    fallback) returns exactly the device projection."""
    from paper_2511_08427_b200 import ops
    from paper_2511_08427_b200.config import PipelineConfig
    from paper_2511_08427_b200.projectors import fp_tensor

    shape, sp = (96, 80, 88), (0.5, 0.5, 0.5)
    cfg = {"geometry_kind": "cone3d", "volume_shape": list(shape), "volume_spacing": list(sp),
           "detector_shape": [128, 136], "detector_spacing": [0.6, 0.6], "number_of_projections": 45,
           "angular_range": 2 * np.pi, "sdd": 1200.0, "sid": 750.0, "step_scale": 0.5}
    if which == 1:
        cfg["number_of_projections"] = 44
    pc = PipelineConfig.from_dict(cfg)
    geom = pc.build_geometry()
    step = pc.sampling().step(geom.volume_spacing)
    x = torch.rand(shape).pin_memory()
    want = fp_tensor(x.cuda(), geom, step).cpu()
    for mode in ("rows", "views"):
        monkeypatch.setenv("TK_FP_PIPE", mode)
        got = ops.py_forward_project(x, pc)
        assert got.is_pinned() and torch.equal(got, want), mode


def test_copy_2d_rows(tk):
    from paper_2511_08427_b200 import ops

    src = torch.rand(7, 24, 33, device="cuda")
    dst = torch.zeros(7, 24, 33).pin_memory()
    s = torch.cuda.current_stream()
    ops._copy_rows(dst, src, 8, 19, s)
    s.synchronize()
    assert torch.equal(dst[:, 8:19], src[:, 8:19].cpu())
    assert float(dst[:, :8].abs().max()) == 0.0 and float(dst[:, 19:].abs().max()) == 0.0
