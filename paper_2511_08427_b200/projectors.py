"""Forward (ray-driven) and back (voxel-driven) projection on the GPU.

Operator API of /root/reference/pkg/src/tomokit/projectors.py (same names,
argument meaning, validation messages and dispatch), executed by the sm_100a
kernels of libtkb200.so.  Two layers:

* tensor level (``fp_*`` / ``bp_*`` / ``*_adjoint``): float32 CUDA tensors in,
  float32 CUDA tensors out, stream-ordered on torch's current stream -- used by
  the autograd Functions, the pipelines and the multi-GPU drivers;
* grid level (``forward_project_*`` / ``back_project_*``): Volume/Sinogram in,
  fresh Volume/Sinogram out, like the reference.

Besides the reference's unmatched pair (ray-driven A, voxel-driven B) this
module exposes the exact transposes A^T and B^T (``transpose_forward_project``,
``transpose_back_project``) for matched adjoints.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .geometry import GeometryCone3D, GeometryFan2D, GeometryParallel2D
from .grids import Sinogram, Volume, as_device_f32

__all__ = [
    "SamplingConfig",
    "forward_project_parallel_2d",
    "back_project_parallel_2d",
    "forward_project_fan_2d",
    "back_project_fan_2d",
    "forward_project_cone_3d",
    "back_project_cone_3d",
    "forward_project",
    "back_project",
    "transpose_forward_project",
    "transpose_back_project",
    "materialize_operator",
    "fp_tensor",
    "bp_tensor",
    "fp_adjoint_tensor",
    "bp_adjoint_tensor",
    "bp_cone_tensor_ex",
]

_MATERIALIZE_LIMIT = 10**7


@dataclass(frozen=True)
class SamplingConfig:
    """Ray-march discretisation: step = step_scale * min(volume spacing)
    (projectors.py:47-62)."""

    step_scale: float = 0.5

    def __post_init__(self):
        if not 0.0 < self.step_scale <= 1.0:
            raise ValueError("step_scale must lie in (0, 1]")

    def step(self, spacing) -> float:
        return self.step_scale * float(min(spacing))


_DEFAULT_CFG = SamplingConfig()


# ---------------------------------------------------------------------------
# tensor level
# ---------------------------------------------------------------------------


def _prep(t: torch.Tensor, shape, what: str) -> torch.Tensor:
    _lib.require_cuda(t, what)
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{what} shape mismatch: got {tuple(t.shape)}, geometry expects {tuple(shape)}")
    if t.dtype != torch.float32:
        t = t.float()
    return t.contiguous()


def _new(shape, like: torch.Tensor) -> torch.Tensor:
    return torch.empty(shape, dtype=torch.float32, device=like.device)


def fp_tensor(vol: torch.Tensor, geom, step: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """Ray-driven forward projection A x of a float32 CUDA volume."""
    vol = _prep(vol, geom.volume_shape, "volume")
    with torch.cuda.device(vol.device):
        s = _lib.stream_ptr(vol.device)
        if isinstance(geom, GeometryCone3D):
            out = _new(geom.sinogram_shape, vol) if out is None else out
            src, minv = geom.ray_constants
            (src, psrc), (minv, pminv) = _lib.host_f64(src), _lib.host_f64(minv)
            nz, ny, nx = geom.volume_shape
            sz, sy, sx = geom.volume_spacing
            rows, cols = geom.detector_shape
            _lib.call("tk_forward_cone_3d", _lib.dev_ptr(vol), nz, ny, nx, sz, sy, sx, psrc, pminv,
                      geom.n_projections, rows, cols, float(step), _lib.dev_ptr(out), s)
            return out
        if isinstance(geom, (GeometryParallel2D,)):
            out = _new(geom.sinogram_shape, vol) if out is None else out
            (c, pc), (sn, ps) = (_lib.host_f64(a) for a in geom.trig)
            ny, nx = geom.volume_shape
            sy, sx = geom.volume_spacing
            if isinstance(geom, GeometryFan2D):
                _lib.call("tk_forward_fan_2d", _lib.dev_ptr(vol), ny, nx, sy, sx, pc, ps,
                          geom.n_projections, geom.sdd, geom.sid, geom.detector_width,
                          geom.detector_spacing, float(step), _lib.dev_ptr(out), s)
            else:
                _lib.call("tk_forward_parallel_2d", _lib.dev_ptr(vol), ny, nx, sy, sx, pc, ps,
                          geom.n_projections, geom.detector_width, geom.detector_spacing,
                          float(step), _lib.dev_ptr(out), s)
            return out
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def fp_bands_tensor(vol: torch.Tensor, geom: GeometryCone3D, step: float, view_offset: int, dests,
                    bands, pitch_rows: int) -> None:
    """Forward projection of ``geom``'s views stored straight into row-band buffers
    (tk_forward_cone_3d_bands): ray (v, r, c) goes to every destination h whose band
    [r0_h, r1_h) holds row r, at ``dests[h][view_offset + v, r - r0_h, c]`` of a
    (V_total, pitch_rows, cols) fp32 buffer.  ``dests`` are device addresses (ints) or
    CUDA tensors -- peer addresses of other GPUs' buffers (CUDA IPC / symmetric memory)
    make the stores the multi-GPU exchange itself."""
    if not isinstance(geom, GeometryCone3D):
        raise TypeError("band-routed forward projection is implemented for cone geometry")
    if len(dests) != len(bands) or not 1 <= len(dests) <= 16:
        raise ValueError("one band per destination, 1 to 16 destinations")
    vol = _prep(vol, geom.volume_shape, "volume")
    ptrs = [int(d.data_ptr()) if isinstance(d, torch.Tensor) else int(d) for d in dests]
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    r0 = (ctypes.c_int * len(bands))(*[int(b[0]) for b in bands])
    r1 = (ctypes.c_int * len(bands))(*[int(b[1]) for b in bands])
    src, minv = geom.ray_constants
    (src, psrc), (minv, pminv) = _lib.host_f64(src), _lib.host_f64(minv)
    nz, ny, nx = geom.volume_shape
    sz, sy, sx = geom.volume_spacing
    rows, cols = geom.detector_shape
    with torch.cuda.device(vol.device):
        _lib.call("tk_forward_cone_3d_bands", _lib.dev_ptr(vol), nz, ny, nx, sz, sy, sx, psrc, pminv,
                  geom.n_projections, rows, cols, float(step), int(view_offset), len(ptrs), arr, r0, r1,
                  int(pitch_rows), _lib.stream_ptr(vol.device))


def forward_kernel_path(geom: GeometryCone3D) -> str:
    """Which cone forward kernel `fp_tensor` runs for this geometry (host-only
    query of tk_forward_cone_3d_path): "mirror" -- one thread marches a ray and
    its z-mirror image (circular orbits) -- or "general"."""
    src, minv = geom.ray_constants
    (src, psrc), (minv, pminv) = _lib.host_f64(src), _lib.host_f64(minv)
    nz, ny, nx = geom.volume_shape
    rows, cols = geom.detector_shape
    lib = _lib.load()
    return "mirror" if lib.tk_forward_cone_3d_path(psrc, pminv, geom.n_projections, rows, cols, nz, ny, nx) \
        else "general"


class ForwardProjectionPlan:
    """A cone-beam volume prepared once (tk_fp_plan_create) and projected in
    view blocks (tk_fp_plan_project) -- used to overlap per-block D2H copies
    with the next block's kernel.  Use as a context manager; the plan's device
    memory is released stream-ordered on the creating stream."""

    def __init__(self, vol: torch.Tensor, geom: GeometryCone3D):
        if not isinstance(geom, GeometryCone3D):
            raise TypeError("forward projection plans are implemented for cone geometry")
        vol = _prep(vol, geom.volume_shape, "volume")
        self.geom, self.device = geom, vol.device
        self._vol = vol  # keep the source alive until the copies are enqueued
        self._handle = ctypes.c_void_p()
        nz, ny, nx = geom.volume_shape
        sz, sy, sx = geom.volume_spacing
        with torch.cuda.device(vol.device):
            self._stream = _lib.stream_ptr(vol.device)
            _lib.call("tk_fp_plan_create", _lib.dev_ptr(vol), nz, ny, nx, sz, sy, sx,
                      ctypes.byref(self._handle), self._stream)

    def project(self, views: slice, out: torch.Tensor, step: float) -> torch.Tensor:
        src, minv = self.geom.ray_constants
        (src, psrc), (minv, pminv) = _lib.host_f64(src[views]), _lib.host_f64(minv[views])
        rows, cols = self.geom.detector_shape
        if tuple(out.shape) != (src.shape[0], rows, cols) or not out.is_contiguous():
            raise ValueError("plan output must be a contiguous (views, rows, cols) tensor")
        with torch.cuda.device(self.device):
            _lib.call("tk_fp_plan_project", self._handle, psrc, pminv, src.shape[0], rows, cols,
                      float(step), _lib.dev_ptr(out), _lib.stream_ptr(self.device))
        return out

    def close(self) -> None:
        if self._handle:
            with torch.cuda.device(self.device):
                _lib.call("tk_fp_plan_destroy", self._handle, self._stream)
            self._handle = ctypes.c_void_p()
            self._vol = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass


def bp_tensor(sino: torch.Tensor, geom, weighted: bool = False,
              out: torch.Tensor | None = None) -> torch.Tensor:
    """Voxel-driven back projection B y (optionally (sid/w)^2-weighted)."""
    sino = _prep(sino, geom.sinogram_shape, "sinogram")
    with torch.cuda.device(sino.device):
        s = _lib.stream_ptr(sino.device)
        out = _new(geom.volume_shape, sino) if out is None else out
        if isinstance(geom, GeometryCone3D):
            mats, pm = _lib.host_f64(geom.matrix_array())
            nz, ny, nx = geom.volume_shape
            sz, sy, sx = geom.volume_spacing
            rows, cols = geom.detector_shape
            _lib.call("tk_back_cone_3d", _lib.dev_ptr(sino), geom.n_projections, rows, cols, pm,
                      geom.sid, int(bool(weighted)), nz, ny, nx, sz, sy, sx, _lib.dev_ptr(out), s)
            return out
        if isinstance(geom, GeometryParallel2D):
            (c, pc), (sn, ps) = (_lib.host_f64(a) for a in geom.trig)
            ny, nx = geom.volume_shape
            sy, sx = geom.volume_spacing
            if isinstance(geom, GeometryFan2D):
                _lib.call("tk_back_fan_2d", _lib.dev_ptr(sino), geom.n_projections,
                          geom.detector_width, pc, ps, geom.sdd, geom.sid, geom.detector_spacing,
                          ny, nx, sy, sx, int(bool(weighted)), _lib.dev_ptr(out), s)
            else:
                if weighted:
                    raise ValueError("parallel backprojection has no distance weighting")
                _lib.call("tk_back_parallel_2d", _lib.dev_ptr(sino), geom.n_projections,
                          geom.detector_width, pc, ps, geom.detector_spacing, ny, nx, sy, sx,
                          _lib.dev_ptr(out), s)
            return out
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def bp_cone_tensor_ex(sino_band: torch.Tensor, geom: GeometryCone3D, weighted: bool, row_begin: int,
                      z_begin: int, z_count: int, out: torch.Tensor | None = None,
                      accumulate: bool = False, views: slice | None = None) -> torch.Tensor:
    """Cone back projection of a z-slab from a detector row band (multi-GPU building block).

    ``sino_band`` is (V', band_rows, cols) holding detector rows
    [row_begin, row_begin + band_rows) of the views selected by ``views``
    (default: all); the result covers global z in [z_begin, z_begin + z_count).
    """
    _lib.require_cuda(sino_band, "sinogram band")
    mats = geom.matrix_array()
    if views is not None:
        mats = mats[views]
    v, band_rows, cols = sino_band.shape
    if v != mats.shape[0] or cols != geom.detector_shape[1]:
        raise ValueError("sinogram band does not match the selected views / detector width")
    nz, ny, nx = geom.volume_shape
    sz, sy, sx = geom.volume_spacing
    sino_band = sino_band.contiguous()
    with torch.cuda.device(sino_band.device):
        if out is None:
            out = (torch.zeros if accumulate else torch.empty)((z_count, ny, nx), dtype=torch.float32,
                                                              device=sino_band.device)
        mats, pm = _lib.host_f64(mats)
        _lib.call("tk_back_cone_3d_ex", _lib.dev_ptr(sino_band), v, geom.detector_shape[0], cols,
                  int(row_begin), band_rows, pm, geom.sid, int(bool(weighted)), nz, ny, nx, sz, sy,
                  sx, int(z_begin), int(z_count), int(bool(accumulate)), _lib.dev_ptr(out),
                  _lib.stream_ptr(sino_band.device))
    return out


def fp_adjoint_tensor(sino: torch.Tensor, geom, step: float, deterministic: bool | None = None) -> torch.Tensor:
    """Exact transpose A^T of the ray-driven forward projector (matched adjoint).

    The scatter sums in fp32 atomics (order-dependent rounding).  ``deterministic``
    (default: ``torch.are_deterministic_algorithms_enabled()``) switches the cone
    transpose to 64-bit fixed-point accumulation: bit-reproducible results."""
    sino = _prep(sino, geom.sinogram_shape, "sinogram")
    if deterministic is None:
        deterministic = torch.are_deterministic_algorithms_enabled()
    with torch.cuda.device(sino.device):
        s = _lib.stream_ptr(sino.device)
        out = _new(geom.volume_shape, sino)
        if isinstance(geom, GeometryCone3D):
            src, minv = geom.ray_constants
            (src, psrc), (minv, pminv) = _lib.host_f64(src), _lib.host_f64(minv)
            nz, ny, nx = geom.volume_shape
            sz, sy, sx = geom.volume_spacing
            rows, cols = geom.detector_shape
            _lib.call("tk_forward_cone_3d_adjoint_ex", _lib.dev_ptr(sino), geom.n_projections, rows,
                      cols, psrc, pminv, nz, ny, nx, sz, sy, sx, float(step), int(bool(deterministic)),
                      _lib.dev_ptr(out), s)
            return out
        if isinstance(geom, GeometryParallel2D):
            _alert_nondeterministic("the 2D forward-projection transpose")
            (c, pc), (sn, ps) = (_lib.host_f64(a) for a in geom.trig)
            ny, nx = geom.volume_shape
            sy, sx = geom.volume_spacing
            if isinstance(geom, GeometryFan2D):
                _lib.call("tk_forward_fan_2d_adjoint", _lib.dev_ptr(sino), geom.n_projections,
                          geom.detector_width, pc, ps, geom.sdd, geom.sid, geom.detector_spacing,
                          float(step), ny, nx, sy, sx, _lib.dev_ptr(out), s)
            else:
                _lib.call("tk_forward_parallel_2d_adjoint", _lib.dev_ptr(sino), geom.n_projections,
                          geom.detector_width, pc, ps, geom.detector_spacing, float(step), ny, nx,
                          sy, sx, _lib.dev_ptr(out), s)
            return out
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def _alert_nondeterministic(what: str) -> None:
    """torch's convention for an op without a deterministic implementation while
    torch.use_deterministic_algorithms(True) is on: raise (or warn if warn_only)."""
    if torch.are_deterministic_algorithms_enabled():
        msg = (f"{what} sums with fp32 atomics and has no deterministic implementation; "
               "use adjoint='paired' or disable torch.use_deterministic_algorithms")
        if torch.is_deterministic_algorithms_warn_only_enabled():
            import warnings

            warnings.warn(msg)
        else:
            raise RuntimeError(msg)


def bp_adjoint_tensor(vol: torch.Tensor, geom, weighted: bool = False) -> torch.Tensor:
    """Exact transpose B^T of the voxel-driven back projector, cone or 2D (fp32
    atomics: summation order not deterministic; raises under torch deterministic mode)."""
    what = "cone" if isinstance(geom, GeometryCone3D) else "2D"
    _alert_nondeterministic(f"the {what} back-projection transpose")
    vol = _prep(vol, geom.volume_shape, "volume")
    with torch.cuda.device(vol.device):
        out = _new(geom.sinogram_shape, vol)
        s = _lib.stream_ptr(vol.device)
        if isinstance(geom, GeometryCone3D):
            mats, pm = _lib.host_f64(geom.matrix_array())
            nz, ny, nx = geom.volume_shape
            sz, sy, sx = geom.volume_spacing
            rows, cols = geom.detector_shape
            _lib.call("tk_back_cone_3d_adjoint", _lib.dev_ptr(vol), nz, ny, nx, sz, sy, sx, pm, geom.sid,
                      int(bool(weighted)), geom.n_projections, rows, cols, _lib.dev_ptr(out), s)
            return out
        if isinstance(geom, GeometryParallel2D):
            (c, pc), (sn, ps) = (_lib.host_f64(a) for a in geom.trig)
            ny, nx = geom.volume_shape
            sy, sx = geom.volume_spacing
            if isinstance(geom, GeometryFan2D):
                _lib.call("tk_back_fan_2d_adjoint", _lib.dev_ptr(vol), ny, nx, sy, sx, pc, ps, geom.n_projections,
                          geom.sdd, geom.sid, geom.detector_width, geom.detector_spacing, int(bool(weighted)),
                          _lib.dev_ptr(out), s)
            else:
                if weighted:
                    raise ValueError("parallel backprojection has no distance weighting")
                _lib.call("tk_back_parallel_2d_adjoint", _lib.dev_ptr(vol), ny, nx, sy, sx, pc, ps,
                          geom.n_projections, geom.detector_width, geom.detector_spacing, _lib.dev_ptr(out), s)
            return out
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


# ---------------------------------------------------------------------------
# grid level (reference API)
# ---------------------------------------------------------------------------


def _require_match(actual, expected, what: str):
    if tuple(actual) != tuple(expected):
        raise ValueError(f"{what} mismatch: got {tuple(actual)}, geometry expects {tuple(expected)}")


def _check_volume(vol: Volume, geom, ndim: int) -> None:
    if vol.data.dim() != ndim:
        raise ValueError(f"expected a {ndim}D volume")
    _require_match(vol.shape, geom.volume_shape, "volume shape")
    _require_match(vol.spacing, geom.volume_spacing, "volume spacing")


def _check_sino(sino: Sinogram, geom) -> None:
    if isinstance(geom, GeometryCone3D):
        if sino.data.dim() != 3:
            raise ValueError("expected a cone-beam sinogram (projections, v, u)")
        _require_match(sino.data.shape, geom.sinogram_shape, "sinogram shape")
        _require_match(sino.detector_spacing, geom.detector_spacing, "detector spacing")
    else:
        if sino.data.dim() != 2:
            raise ValueError("expected a 2D-geometry sinogram (projections, u)")
        _require_match(sino.data.shape, geom.sinogram_shape, "sinogram shape")
        _require_match(sino.detector_spacing, (geom.detector_spacing,), "detector spacing")


def _det_spacing(geom) -> tuple:
    return geom.detector_spacing if isinstance(geom, GeometryCone3D) else (geom.detector_spacing,)


def forward_project_parallel_2d(vol: Volume, geom: GeometryParallel2D,
                                cfg: SamplingConfig = _DEFAULT_CFG) -> Sinogram:
    _check_volume(vol, geom, 2)
    return Sinogram(fp_tensor(vol.data, geom, cfg.step(geom.volume_spacing)), _det_spacing(geom))


def back_project_parallel_2d(sino: Sinogram, geom: GeometryParallel2D) -> Volume:
    _check_sino(sino, geom)
    return Volume(bp_tensor(sino.data, geom, False), geom.volume_spacing)


def forward_project_fan_2d(vol: Volume, geom: GeometryFan2D,
                           cfg: SamplingConfig = _DEFAULT_CFG) -> Sinogram:
    _check_volume(vol, geom, 2)
    return Sinogram(fp_tensor(vol.data, geom, cfg.step(geom.volume_spacing)), _det_spacing(geom))


def back_project_fan_2d(sino: Sinogram, geom: GeometryFan2D, fdk_weighting: bool = False) -> Volume:
    _check_sino(sino, geom)
    return Volume(bp_tensor(sino.data, geom, bool(fdk_weighting)), geom.volume_spacing)


def forward_project_cone_3d(vol: Volume, geom: GeometryCone3D,
                            cfg: SamplingConfig = _DEFAULT_CFG) -> Sinogram:
    _check_volume(vol, geom, 3)
    geom.ray_constants  # validates the matrices (degenerate M) before launching
    return Sinogram(fp_tensor(vol.data, geom, cfg.step(geom.volume_spacing)), geom.detector_spacing)


def back_project_cone_3d(sino: Sinogram, geom: GeometryCone3D, fdk_weighting: bool = False) -> Volume:
    _check_sino(sino, geom)
    return Volume(bp_tensor(sino.data, geom, bool(fdk_weighting)), geom.volume_spacing)


def forward_project(vol: Volume, geom, cfg: SamplingConfig = _DEFAULT_CFG) -> Sinogram:
    """Geometry-dispatching forward projection (projectors.py:251-259)."""
    if isinstance(geom, GeometryCone3D):
        return forward_project_cone_3d(vol, geom, cfg)
    if isinstance(geom, GeometryFan2D):
        return forward_project_fan_2d(vol, geom, cfg)
    if isinstance(geom, GeometryParallel2D):
        return forward_project_parallel_2d(vol, geom, cfg)
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def back_project(sino: Sinogram, geom, fdk_weighting: bool = False) -> Volume:
    """Geometry-dispatching back projection (projectors.py:262-272)."""
    if isinstance(geom, GeometryCone3D):
        return back_project_cone_3d(sino, geom, fdk_weighting)
    if isinstance(geom, GeometryFan2D):
        return back_project_fan_2d(sino, geom, fdk_weighting)
    if isinstance(geom, GeometryParallel2D):
        if fdk_weighting:
            raise ValueError("parallel backprojection has no distance weighting")
        return back_project_parallel_2d(sino, geom)
    raise TypeError(f"unsupported geometry {type(geom).__name__}")


def transpose_forward_project(sino: Sinogram, geom, cfg: SamplingConfig = _DEFAULT_CFG) -> Volume:
    """Exact A^T (matched adjoint of the ray-driven forward projector)."""
    if not isinstance(geom, (GeometryCone3D, GeometryParallel2D)):
        raise TypeError(f"unsupported geometry {type(geom).__name__}")
    _check_sino(sino, geom)
    return Volume(fp_adjoint_tensor(sino.data, geom, cfg.step(geom.volume_spacing)), geom.volume_spacing)


def transpose_back_project(vol: Volume, geom, fdk_weighting: bool = False) -> Sinogram:
    """Exact B^T (matched adjoint of the voxel-driven back projector: cone, fan or parallel)."""
    _check_volume(vol, geom, 3 if isinstance(geom, GeometryCone3D) else 2)
    spacing = geom.detector_spacing if isinstance(geom, GeometryCone3D) else (geom.detector_spacing,)
    return Sinogram(bp_adjoint_tensor(vol.data, geom, fdk_weighting), spacing)


def _sizes(geom):
    n_vox = int(np.prod(geom.volume_shape))
    return n_vox, int(np.prod(geom.sinogram_shape))


def materialize_operator(geom, cfg: SamplingConfig = _DEFAULT_CFG, which: str = "forward") -> np.ndarray:
    """Dense float64 matrix of an operator, one unit impulse per column
    (projectors.py:294-324).  Test-scale only (<= 1e7 entries)."""
    n_vox, n_meas = _sizes(geom)
    if n_vox * n_meas > _MATERIALIZE_LIMIT:
        raise ValueError(f"operator too large to materialize: {n_vox} x {n_meas} > {_MATERIALIZE_LIMIT}")
    dev = torch.device("cuda", torch.cuda.current_device())
    if which == "forward":
        mat = np.empty((n_meas, n_vox))
        imp = torch.zeros(n_vox, dtype=torch.float32, device=dev)
        for j in range(n_vox):
            imp.zero_()
            imp[j] = 1.0
            mat[:, j] = fp_tensor(imp.view(geom.volume_shape), geom,
                                  cfg.step(geom.volume_spacing)).double().cpu().numpy().ravel()
        return mat
    if which == "back":
        mat = np.empty((n_vox, n_meas))
        imp = torch.zeros(n_meas, dtype=torch.float32, device=dev)
        for j in range(n_meas):
            imp.zero_()
            imp[j] = 1.0
            mat[:, j] = bp_tensor(imp.view(geom.sinogram_shape), geom).double().cpu().numpy().ravel()
        return mat
    raise ValueError("which must be 'forward' or 'back'")
