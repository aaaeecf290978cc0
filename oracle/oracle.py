"""CPU ORACLE -- test infrastructure only (never the product path).

A float64 restatement of the reference CT-operator path
(/root/reference/pkg/src/tomokit).  The O(N_vox * N_views) kernels live in
``tk_oracle.c`` (plain C + OpenMP, loaded here with ctypes); the O(N_views)
geometry and O(sinogram) filtering host logic is restated below in numpy.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.

Parity of this oracle with the reference itself is pinned by
``tests/test_oracle_golden.py`` against ``tests/golden/*.npz``, which
``tests/golden/make_golden.py`` produced by importing the reference in the
build container.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "libtk_oracle.so"
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int
_F = ctypes.c_double

_SIGS = {
    "ora_forward_parallel_2d": [_D, _I, _I, _F, _F, _D, _D, _I, _I, _F, _F, _D],
    "ora_back_parallel_2d": [_D, _I, _I, _D, _D, _F, _I, _I, _F, _F, _D],
    "ora_forward_fan_2d": [_D, _I, _I, _F, _F, _D, _D, _I, _F, _F, _I, _F, _F, _D],
    "ora_back_fan_2d": [_D, _I, _I, _D, _D, _F, _F, _F, _I, _I, _F, _F, _I, _D],
    "ora_forward_cone_3d": [_D, _I, _I, _I, _F, _F, _F, _D, _D, _I, _I, _I, _F, _D],
    "ora_back_cone_3d": [_D, _I, _I, _I, _D, _F, _I, _I, _I, _I, _F, _F, _F, _D],
    "ora_forward_parallel_2d_transpose": [_D, _I, _I, _F, _F, _D, _D, _I, _I, _F, _F, _D],
    "ora_forward_fan_2d_transpose": [_D, _I, _I, _F, _F, _D, _D, _I, _F, _F, _I, _F, _F, _D],
    "ora_forward_cone_3d_transpose": [_D, _I, _I, _I, _F, _F, _F, _D, _D, _I, _I, _I, _F, _D],
    "ora_back_cone_3d_transpose": [_D, _I, _I, _I, _D, _F, _I, _I, _I, _I, _F, _F, _F, _D],
    "ora_back_parallel_2d_transpose": [_D, _I, _I, _D, _D, _F, _I, _I, _F, _F, _D],
    "ora_back_fan_2d_transpose": [_D, _I, _I, _D, _D, _F, _F, _F, _I, _I, _F, _F, _I, _D],
    "ora_num_threads": [],
    "ora_set_num_threads": [_I],
}


def build() -> Path:
    """Compile tk_oracle.c with the committed Makefile (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists() or _LIB_PATH.stat().st_mtime < (_HERE / "tk_oracle.c").stat().st_mtime:
            build()
        handle = ctypes.CDLL(str(_LIB_PATH))
        for name, args in _SIGS.items():
            fn = getattr(handle, name)
            fn.argtypes = args
            fn.restype = _I if name == "ora_num_threads" else None
        _lib = handle
    return _lib


def num_threads() -> int:
    return int(lib().ora_num_threads())


def set_num_threads(n: int) -> None:
    lib().ora_set_num_threads(int(n))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# Geometry restatement (reference geometry.py / projectors.py host logic)
# ---------------------------------------------------------------------------


def circular_angles(n: int, angular_range: float) -> np.ndarray:
    """geometry.py:240-248 -- i * range / n, endpoint excluded."""
    return np.arange(int(n)) * (float(angular_range) / int(n))


def pose_matrix(src, center, u_dir, v_dir, detector_shape, detector_spacing) -> np.ndarray:
    """geometry.py:251-281 (pose_to_projection_matrix) with Pose.normal (93-99)."""
    rows, cols = (int(n) for n in detector_shape)
    dv, du = (float(s) for s in detector_spacing)
    s = _f64(src)
    c = _f64(center)
    u = _f64(u_dir)
    v = _f64(v_dir)
    n = np.cross(u, v)
    if float((c - s) @ n) < 0:
        n = -n
    depth = float((c - s) @ n)
    off = c - s
    m = np.empty((3, 4))
    m[0, :3] = (depth / du) * u + ((cols - 1) / 2.0 - float(off @ u) / du) * n
    m[1, :3] = (depth / dv) * v + ((rows - 1) / 2.0 - float(off @ v) / dv) * n
    m[2, :3] = n
    m[:, 3] = -m[:, :3] @ s
    return m


def circular_pose(theta: float, sdd: float, sid: float):
    """geometry.py:284-292."""
    ct, st = np.cos(theta), np.sin(theta)
    return (
        np.array([sid * ct, sid * st, 0.0]),
        np.array([-(sdd - sid) * ct, -(sdd - sid) * st, 0.0]),
        np.array([-st, ct, 0.0]),
        np.array([0.0, 0.0, 1.0]),
    )


def circular_matrices(n, angular_range, sdd, sid, detector_shape, detector_spacing) -> np.ndarray:
    """geometry.py:295-312 -> (V, 3, 4)."""
    return np.stack(
        [
            pose_matrix(*circular_pose(t, float(sdd), float(sid)), detector_shape, detector_spacing)
            for t in circular_angles(n, angular_range)
        ]
    )


def normalize_raw(m) -> np.ndarray:
    """geometry.py:117-131 (ProjectionMatrix.from_raw)."""
    m = _f64(m).reshape(3, 4)
    norm = float(np.linalg.norm(m[2, :3]))
    if m[2, 3] < 0:
        norm = -norm
    return m / norm


def cone_rays(mats: np.ndarray):
    """projectors.py:191-202 with geometry.py:133-139 (source = SVD null vector)."""
    mats = _f64(mats)
    n = mats.shape[0]
    sources = np.empty((n, 3))
    minv = np.empty((n, 3, 3))
    for i in range(n):
        m = mats[i, :, :3]
        if abs(np.linalg.det(m)) < 1e-12:
            raise ValueError(f"projection matrix {i} is degenerate (singular M block)")
        _, _, vh = np.linalg.svd(mats[i])
        h = vh[-1]
        sources[i] = h[:3] / h[3]
        minv[i] = np.linalg.inv(m)
    return sources, minv


def step_of(spacing, step_scale: float = 0.5) -> float:
    """projectors.py:61-62 (SamplingConfig.step)."""
    return float(step_scale) * float(min(spacing))


# ---------------------------------------------------------------------------
# Kernels (C, float64).  Inputs are UNPADDED; padding restates projectors.py:26-29.
# ---------------------------------------------------------------------------


def forward_parallel_2d(vol, spacing, angles, n_det, ds, step) -> np.ndarray:
    volp = _f64(np.pad(_f64(vol), 1))
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    out = np.empty((ang.size, int(n_det)))
    lib().ora_forward_parallel_2d(_p(volp), volp.shape[0], volp.shape[1], float(spacing[0]),
                                  float(spacing[1]), _p(c), _p(s), ang.size, int(n_det),
                                  float(ds), float(step), _p(out))
    return out


def back_parallel_2d(sino, angles, ds, volume_shape, spacing) -> np.ndarray:
    sino = _f64(sino)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    ny, nx = (int(n) for n in volume_shape)
    out = np.empty((ny, nx))
    lib().ora_back_parallel_2d(_p(sino), sino.shape[0], sino.shape[1], _p(c), _p(s), float(ds),
                               ny, nx, float(spacing[0]), float(spacing[1]), _p(out))
    return out


def forward_fan_2d(vol, spacing, angles, sdd, sid, n_det, ds, step) -> np.ndarray:
    volp = _f64(np.pad(_f64(vol), 1))
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    out = np.empty((ang.size, int(n_det)))
    lib().ora_forward_fan_2d(_p(volp), volp.shape[0], volp.shape[1], float(spacing[0]),
                             float(spacing[1]), _p(c), _p(s), ang.size, float(sdd), float(sid),
                             int(n_det), float(ds), float(step), _p(out))
    return out


def back_fan_2d(sino, angles, sdd, sid, ds, volume_shape, spacing, weighted=False) -> np.ndarray:
    sino = _f64(sino)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    ny, nx = (int(n) for n in volume_shape)
    out = np.empty((ny, nx))
    lib().ora_back_fan_2d(_p(sino), sino.shape[0], sino.shape[1], _p(c), _p(s), float(sdd),
                          float(sid), float(ds), ny, nx, float(spacing[0]), float(spacing[1]),
                          int(bool(weighted)), _p(out))
    return out


def forward_cone_3d(vol, spacing, mats, detector_shape, step) -> np.ndarray:
    volp = _f64(np.pad(_f64(vol), 1))
    sources, minv = cone_rays(mats)
    rows, cols = (int(n) for n in detector_shape)
    nv = sources.shape[0]
    out = np.empty((nv, rows, cols))
    lib().ora_forward_cone_3d(_p(volp), *volp.shape, float(spacing[0]), float(spacing[1]),
                              float(spacing[2]), _p(_f64(sources)), _p(_f64(minv)), nv, rows,
                              cols, float(step), _p(out))
    return out


def back_cone_3d(sino, mats, sid, volume_shape, spacing, weighted=False) -> np.ndarray:
    sino = _f64(sino)
    mats = _f64(mats)
    nz, ny, nx = (int(n) for n in volume_shape)
    out = np.empty((nz, ny, nx))
    lib().ora_back_cone_3d(_p(sino), sino.shape[0], sino.shape[1], sino.shape[2], _p(mats),
                           float(sid), int(bool(weighted)), nz, ny, nx, float(spacing[0]),
                           float(spacing[1]), float(spacing[2]), _p(out))
    return out


def forward_parallel_2d_T(sino, volume_shape, spacing, angles, ds, step) -> np.ndarray:
    """Exact transpose of forward_parallel_2d (matched adjoint oracle)."""
    sino = _f64(sino)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    ny, nx = (int(n) for n in volume_shape)
    adjp = np.empty((ny + 2, nx + 2))
    lib().ora_forward_parallel_2d_transpose(_p(sino), ny + 2, nx + 2, float(spacing[0]),
                                            float(spacing[1]), _p(c), _p(s), ang.size,
                                            sino.shape[1], float(ds), float(step), _p(adjp))
    return adjp[1:-1, 1:-1].copy()


def forward_fan_2d_T(sino, volume_shape, spacing, angles, sdd, sid, ds, step) -> np.ndarray:
    sino = _f64(sino)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    ny, nx = (int(n) for n in volume_shape)
    adjp = np.empty((ny + 2, nx + 2))
    lib().ora_forward_fan_2d_transpose(_p(sino), ny + 2, nx + 2, float(spacing[0]),
                                       float(spacing[1]), _p(c), _p(s), ang.size, float(sdd),
                                       float(sid), sino.shape[1], float(ds), float(step), _p(adjp))
    return adjp[1:-1, 1:-1].copy()


def forward_cone_3d_T(sino, volume_shape, spacing, mats, step) -> np.ndarray:
    sino = _f64(sino)
    sources, minv = cone_rays(mats)
    nz, ny, nx = (int(n) for n in volume_shape)
    adjp = np.empty((nz + 2, ny + 2, nx + 2))
    lib().ora_forward_cone_3d_transpose(_p(sino), nz + 2, ny + 2, nx + 2, float(spacing[0]),
                                        float(spacing[1]), float(spacing[2]), _p(_f64(sources)),
                                        _p(_f64(minv)), sources.shape[0], sino.shape[1],
                                        sino.shape[2], float(step), _p(adjp))
    return adjp[1:-1, 1:-1, 1:-1].copy()


def back_cone_3d_T(vol, mats, sid, detector_shape, spacing, weighted=False) -> np.ndarray:
    vol = _f64(vol)
    mats = _f64(mats)
    rows, cols = (int(n) for n in detector_shape)
    nz, ny, nx = vol.shape
    out = np.empty((mats.shape[0], rows, cols))
    lib().ora_back_cone_3d_transpose(_p(vol), mats.shape[0], rows, cols, _p(mats), float(sid),
                                     int(bool(weighted)), nz, ny, nx, float(spacing[0]),
                                     float(spacing[1]), float(spacing[2]), _p(out))
    return out


def back_parallel_2d_T(img, angles, ds, n_det, spacing) -> np.ndarray:
    """Exact transpose of back_parallel_2d (_kernels.py:174-195)."""
    img = _f64(img)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    out = np.empty((ang.size, int(n_det)))
    lib().ora_back_parallel_2d_transpose(_p(img), ang.size, int(n_det), _p(c), _p(s), float(ds), img.shape[0],
                                         img.shape[1], float(spacing[0]), float(spacing[1]), _p(out))
    return out


def back_fan_2d_T(img, angles, sdd, sid, ds, n_det, spacing, weighted=False) -> np.ndarray:
    """Exact transpose of back_fan_2d (_kernels.py:219-251)."""
    img = _f64(img)
    ang = _f64(angles)
    c, s = _f64(np.cos(ang)), _f64(np.sin(ang))
    out = np.empty((ang.size, int(n_det)))
    lib().ora_back_fan_2d_transpose(_p(img), ang.size, int(n_det), _p(c), _p(s), float(sdd), float(sid),
                                    float(ds), img.shape[0], img.shape[1], float(spacing[0]), float(spacing[1]),
                                    int(bool(weighted)), _p(out))
    return out


# ---------------------------------------------------------------------------
# Filters (reference filters.py), numpy float64
# ---------------------------------------------------------------------------


def pad_length(width: int) -> int:
    """filters.py:83-87."""
    n = 1
    while n < 2 * int(width):
        n *= 2
    return n


def ramp_weights(width: int, spacing: float) -> np.ndarray:
    """filters.py:90-110."""
    n_pad = pad_length(width)
    kernel = np.zeros(n_pad)
    kernel[0] = 1.0 / (4.0 * spacing**2)
    odd = np.arange(1, n_pad // 2 + 1, 2)
    vals = -1.0 / (np.pi * odd * spacing) ** 2
    kernel[odd] = vals
    kernel[n_pad - odd] = vals
    w = np.fft.fft(kernel).real
    w = np.maximum(w, 0.0)
    w = 0.5 * (w + np.roll(w[::-1], 1))
    w[0] = 0.0
    return w


def _bin_fractions(n_pad: int) -> np.ndarray:
    """filters.py:118-121."""
    k = np.minimum(np.arange(n_pad), n_pad - np.arange(n_pad))
    return k / n_pad


def filter_weights(kind: str, width: int, spacing: float) -> np.ndarray:
    """filters.py:113-133 (ramp / shepp_logan / cosine)."""
    w = ramp_weights(width, spacing)
    if kind == "ramp":
        return w
    if kind == "shepp_logan":
        return w * np.sinc(_bin_fractions(w.size))
    if kind == "cosine":
        return w * np.cos(np.pi * _bin_fractions(w.size))
    raise ValueError(kind)


def fft_filter(data, weights, spacing) -> np.ndarray:
    """filters.py:136-151."""
    data = _f64(data)
    width = data.shape[-1]
    n_pad = weights.size
    half = weights[: n_pad // 2 + 1]
    spec = np.fft.rfft(data, n=n_pad, axis=-1)
    return np.fft.irfft(spec * half, n=n_pad, axis=-1)[..., :width] * float(spacing)


def cosine_preweight_cone(sino, sdd, detector_spacing) -> np.ndarray:
    """filters.py:154-165."""
    sino = _f64(sino)
    rows, cols = sino.shape[1:]
    dv, du = detector_spacing
    u = (np.arange(cols) - (cols - 1) / 2.0) * du
    v = (np.arange(rows) - (rows - 1) / 2.0) * dv
    w = sdd / np.sqrt(sdd**2 + u[np.newaxis, :] ** 2 + v[:, np.newaxis] ** 2)
    return sino * w


def preweight_fan(sino, sdd, ds) -> np.ndarray:
    """filters.py:168-171."""
    sino = _f64(sino)
    u = (np.arange(sino.shape[-1]) - (sino.shape[-1] - 1) / 2.0) * ds
    return sino * (sdd / np.sqrt(sdd**2 + u**2))


def round_stage(data) -> np.ndarray:
    """filters.py:174-177."""
    return np.asarray(data).astype(np.float32).astype(np.float64)


def filter_stage_cone(sino, sdd, sid, detector_spacing, kind="ramp") -> np.ndarray:
    """filters.py:204-211 + 180-201 for cone geometry."""
    pre = cosine_preweight_cone(sino, sdd, detector_spacing)
    du = detector_spacing[1]
    pitch = du * sid / sdd
    w = filter_weights(kind, sino.shape[-1], pitch)
    return round_stage(fft_filter(pre, w, pitch))


def filter_stage_fan(sino, sdd, sid, ds, kind="ramp") -> np.ndarray:
    pre = preweight_fan(sino, sdd, ds)
    pitch = ds * sid / sdd
    w = filter_weights(kind, np.asarray(sino).shape[-1], pitch)
    return round_stage(fft_filter(pre, w, pitch))


def filter_stage_parallel(sino, ds, kind="ramp") -> np.ndarray:
    w = filter_weights(kind, np.asarray(sino).shape[-1], ds)
    return round_stage(fft_filter(sino, w, ds))


def fdk_cone_3d(sino, mats, sdd, sid, detector_spacing, volume_shape, spacing, kind="ramp"):
    """filters.py:214-219 + 233-236."""
    f = filter_stage_cone(sino, sdd, sid, detector_spacing, kind)
    vol = back_cone_3d(f, mats, sid, volume_shape, spacing, weighted=True)
    return round_stage(vol * (np.pi / np.asarray(mats).shape[0]))


def fbp_parallel_2d(sino, angles, ds, volume_shape, spacing, kind="ramp"):
    f = filter_stage_parallel(sino, ds, kind)
    vol = back_parallel_2d(f, angles, ds, volume_shape, spacing)
    return round_stage(vol * (np.pi / np.asarray(angles).size))


def fbp_fan_2d(sino, angles, sdd, sid, ds, volume_shape, spacing, kind="ramp"):
    f = filter_stage_fan(sino, sdd, sid, ds, kind)
    vol = back_fan_2d(f, angles, sdd, sid, ds, volume_shape, spacing, weighted=True)
    return round_stage(vol * (np.pi / np.asarray(angles).size))


# ---------------------------------------------------------------------------
# Phantoms (reference phantoms.py) -- synthetic-input generator for checks
# ---------------------------------------------------------------------------

SHEPP_LOGAN_3D = (
    (1.00, 0.6900, 0.9200, 0.810, 0.00, 0.0000, 0.000, 0.0),
    (-0.80, 0.6624, 0.8740, 0.780, 0.00, -0.0184, 0.000, 0.0),
    (-0.20, 0.1100, 0.3100, 0.220, 0.22, 0.0000, 0.000, -18.0),
    (-0.20, 0.1600, 0.4100, 0.280, -0.22, 0.0000, 0.000, 18.0),
    (0.10, 0.2100, 0.2500, 0.410, 0.00, 0.3500, -0.150, 0.0),
    (0.10, 0.0460, 0.0460, 0.050, 0.00, 0.1000, 0.250, 0.0),
    (0.10, 0.0460, 0.0460, 0.050, 0.00, -0.1000, 0.250, 0.0),
    (0.10, 0.0460, 0.0230, 0.050, -0.08, -0.6050, 0.000, 0.0),
    (0.10, 0.0230, 0.0230, 0.020, 0.00, -0.6050, 0.000, 0.0),
    (0.10, 0.0230, 0.0460, 0.020, 0.06, -0.6050, 0.000, 0.0),
)


def shepp_logan_3d(shape) -> np.ndarray:
    """phantoms.py:118-133 (hard membership at voxel centres)."""
    nz, ny, nx = (int(n) for n in shape)
    ax = lambda n: (np.arange(n) - (n - 1) / 2.0) * (2.0 / n)  # noqa: E731
    x = ax(nx)[None, None, :]
    y = ax(ny)[None, :, None]
    z = ax(nz)[:, None, None]
    vol = np.zeros((nz, ny, nx))
    for delta, a, b, c, x0, y0, z0, phi_deg in SHEPP_LOGAN_3D:
        phi = np.deg2rad(phi_deg)
        dx, dy, dz = x - x0, y - y0, z - z0
        xr = dx * np.cos(phi) + dy * np.sin(phi)
        yr = -dx * np.sin(phi) + dy * np.cos(phi)
        vol[(xr / a) ** 2 + (yr / b) ** 2 + (dz / c) ** 2 <= 1.0] += delta
    return vol


def rel_l2(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = float(np.linalg.norm(want))
    return float(np.linalg.norm(got - want)) / (den if den > 0 else 1.0)


if os.environ.get("TK_ORACLE_THREADS"):
    set_num_threads(int(os.environ["TK_ORACLE_THREADS"]))
