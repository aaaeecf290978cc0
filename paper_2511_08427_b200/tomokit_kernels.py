"""Kernel-level drop-in for the reference: the six numba kernels of
``tomokit._kernels`` (/root/reference/pkg/src/tomokit/_kernels.py:160-322) and
the numpy row filter ``tomokit.filters.fft_filter`` (filters.py:136-151),
re-implemented on libtkb200.so with the reference's exact signatures and
calling conventions: float64 numpy arrays in, caller-allocated ``out``
overwritten, the forward kernels receiving the one-voxel zero-padded volume
(projectors.py:26-29; stripped here, the library zero-extends internally).

This is the module INTEGRATION.md section 1 describes: a maintainer binds it
with ``install(tomokit)``, which rebinds the module attributes the reference's
call sites use (``projectors.py`` calls ``_kernels.<name>(...)``), so every
layer above -- projectors, filters, autodiff, the tomokit_layers boundary, the
CLI -- runs on the GPU unchanged.  Grids cross as float32 (the reference's own
boundary precision, tomokit_layers/ops.py:57-69); results are widened back to
the caller's float64 buffers.  No CPU fallback: without a CUDA device every
call raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

__all__ = ["forward_parallel_2d", "back_parallel_2d", "forward_fan_2d", "back_fan_2d", "forward_cone_3d",
           "back_cone_3d", "fft_filter", "warmup", "install"]


def _dev(a: np.ndarray) -> torch.Tensor:
    if not torch.cuda.is_available():
        raise RuntimeError("tomokit_kernels: no CUDA device (libtkb200 has no CPU path)")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _unpad(volp: np.ndarray) -> np.ndarray:
    return volp[(slice(1, -1),) * volp.ndim]


def _store(out: np.ndarray, t: torch.Tensor) -> None:
    out[...] = t.cpu().numpy()


def _stream():
    return _lib.stream_ptr(torch.device("cuda", torch.cuda.current_device()))


def forward_parallel_2d(volp, sy, sx, cos_a, sin_a, n_det, ds, step, out):
    """_kernels.py:160-171."""
    vol = _dev(_unpad(volp))
    ny, nx = vol.shape
    (c, pc), (s, ps) = _lib.host_f64(cos_a), _lib.host_f64(sin_a)
    res = torch.empty((c.shape[0], int(n_det)), dtype=torch.float32, device="cuda")
    _lib.call("tk_forward_parallel_2d", _lib.dev_ptr(vol), ny, nx, float(sy), float(sx), pc, ps, c.shape[0],
              int(n_det), float(ds), float(step), _lib.dev_ptr(res), _stream())
    _store(out, res)


def back_parallel_2d(sino, cos_a, sin_a, ds, ny, nx, sy, sx, out):
    """_kernels.py:174-195."""
    y = _dev(sino)
    (c, pc), (s, ps) = _lib.host_f64(cos_a), _lib.host_f64(sin_a)
    res = torch.empty((int(ny), int(nx)), dtype=torch.float32, device="cuda")
    _lib.call("tk_back_parallel_2d", _lib.dev_ptr(y), y.shape[0], y.shape[1], pc, ps, float(ds), int(ny), int(nx),
              float(sy), float(sx), _lib.dev_ptr(res), _stream())
    _store(out, res)


def forward_fan_2d(volp, sy, sx, cos_a, sin_a, sdd, sid, n_det, ds, step, out):
    """_kernels.py:198-216."""
    vol = _dev(_unpad(volp))
    ny, nx = vol.shape
    (c, pc), (s, ps) = _lib.host_f64(cos_a), _lib.host_f64(sin_a)
    res = torch.empty((c.shape[0], int(n_det)), dtype=torch.float32, device="cuda")
    _lib.call("tk_forward_fan_2d", _lib.dev_ptr(vol), ny, nx, float(sy), float(sx), pc, ps, c.shape[0],
              float(sdd), float(sid), int(n_det), float(ds), float(step), _lib.dev_ptr(res), _stream())
    _store(out, res)


def back_fan_2d(sino, cos_a, sin_a, sdd, sid, ds, ny, nx, sy, sx, weighted, out):
    """_kernels.py:219-251."""
    y = _dev(sino)
    (c, pc), (s, ps) = _lib.host_f64(cos_a), _lib.host_f64(sin_a)
    res = torch.empty((int(ny), int(nx)), dtype=torch.float32, device="cuda")
    _lib.call("tk_back_fan_2d", _lib.dev_ptr(y), y.shape[0], y.shape[1], pc, ps, float(sdd), float(sid),
              float(ds), int(ny), int(nx), float(sy), float(sx), int(bool(weighted)), _lib.dev_ptr(res), _stream())
    _store(out, res)


def forward_cone_3d(volp, sz, sy, sx, sources, minv, rows, cols, step, out):
    """_kernels.py:254-278 (sources, minv: projectors._cone_rays, projectors.py:191-202)."""
    vol = _dev(_unpad(volp))
    nz, ny, nx = vol.shape
    (src, psrc), (mi, pmi) = _lib.host_f64(sources), _lib.host_f64(minv)
    res = torch.empty((src.shape[0], int(rows), int(cols)), dtype=torch.float32, device="cuda")
    _lib.call("tk_forward_cone_3d", _lib.dev_ptr(vol), nz, ny, nx, float(sz), float(sy), float(sx), psrc, pmi,
              src.shape[0], int(rows), int(cols), float(step), _lib.dev_ptr(res), _stream())
    _store(out, res)


def back_cone_3d(sino, mats, sid, weighted, nz, ny, nx, sz, sy, sx, out):
    """_kernels.py:281-322."""
    y = _dev(sino)
    m, pm = _lib.host_f64(mats)
    res = torch.empty((int(nz), int(ny), int(nx)), dtype=torch.float32, device="cuda")
    _lib.call("tk_back_cone_3d", _lib.dev_ptr(y), y.shape[0], y.shape[1], y.shape[2], pm, float(sid),
              int(bool(weighted)), int(nz), int(ny), int(nx), float(sz), float(sy), float(sx), _lib.dev_ptr(res),
              _stream())
    _store(out, res)


def fft_filter(sino, filt):
    """filters.py:136-151 on the GPU row filter (tk_fft_filter_rows, no pre-weight):
    the same padding check and message, the same Sinogram result type."""
    from tomokit.grids import Sinogram  # the caller's container type

    data = np.asarray(sino.data)
    width = data.shape[-1]
    if filt.n_pad < 2 * width:
        raise ValueError(f"filter padding {filt.n_pad} too short for detector width {width}")
    half, ph = _lib.host_f64(np.asarray(filt.weights, np.float64)[: filt.n_pad // 2 + 1])
    x = _dev(data.reshape(-1, width))
    res = torch.empty_like(x)
    det_rows = data.shape[-2] if data.ndim == 3 else 1
    _lib.call("tk_fft_filter_rows", _lib.dev_ptr(x), x.shape[0], width, det_rows, ph, int(filt.n_pad),
              float(filt.detector_spacing), 0.0, 1.0, 1.0, _lib.dev_ptr(res), _stream())
    return Sinogram(res.cpu().numpy().astype(np.float64).reshape(data.shape), sino.detector_spacing)


def warmup():
    """_kernels.warmup (_kernels.py:325-346): loads the library and touches the device."""
    _lib.load()
    torch.zeros(1, device="cuda")


def install(tomokit_module) -> list:
    """Rebind the reference's kernel layer (and row filter) to this module: every
    attribute of a loaded ``tomokit*`` module that IS one of the replaced
    functions (``_kernels.<name>``, ``filters.fft_filter`` and names imported
    from them, e.g. ``autodiff.fft_filter``).  Returns (module, name, original)
    triples so the binding can be undone."""
    import importlib
    import sys

    root = tomokit_module.__name__
    kernels = importlib.import_module(root + "._kernels")
    filters = importlib.import_module(root + ".filters")
    for sub in ("projectors", "autodiff", "cli", "config"):
        try:
            importlib.import_module(f"{root}.{sub}")
        except ImportError:
            pass
    originals = {getattr(kernels, n): globals()[n] for n in
                 ("forward_parallel_2d", "back_parallel_2d", "forward_fan_2d", "back_fan_2d", "forward_cone_3d",
                  "back_cone_3d", "warmup")}
    originals[filters.fft_filter] = fft_filter
    saved = []
    for mname, mod in list(sys.modules.items()):
        if mod is None or not (mname == root or mname.startswith(root + ".")):
            continue
        for attr, val in list(vars(mod).items()):
            try:
                new = originals.get(val)
            except TypeError:  # unhashable attribute
                continue
            if new is not None:
                saved.append((mod, attr, val))
                setattr(mod, attr, new)
    return saved
