"""ctypes binding of libtkb200.so (the sm_100a kernels behind include/tk_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
operator raises.  Grids cross the ABI as raw device pointers of torch tensors;
per-view geometry as host float64 numpy arrays; the stream is torch's current
CUDA stream, so the kernels order correctly with surrounding torch work.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import numpy as np
import torch

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libtkb200.so"

_c_int = ctypes.c_int
_c_ll = ctypes.c_longlong
_c_dbl = ctypes.c_double
_ptr = ctypes.c_void_p
_dptr = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (restype int unless noted); mirrors include/tk_b200.h
SIGNATURES = {
    "tk_version": [],
    "tk_last_error": [],
    "tk_device_info": [ctypes.POINTER(_c_int)] * 3,
    "tk_launch_count": [],
    "tk_cached_bytes": [],
    "tk_release_cached_memory": [],
    "tk_forward_parallel_2d": [_ptr, _c_int, _c_int, _c_dbl, _c_dbl, _dptr, _dptr, _c_int, _c_int,
                               _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_back_parallel_2d": [_ptr, _c_int, _c_int, _dptr, _dptr, _c_dbl, _c_int, _c_int, _c_dbl,
                            _c_dbl, _ptr, _ptr],
    "tk_forward_fan_2d": [_ptr, _c_int, _c_int, _c_dbl, _c_dbl, _dptr, _dptr, _c_int, _c_dbl, _c_dbl,
                          _c_int, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_back_fan_2d": [_ptr, _c_int, _c_int, _dptr, _dptr, _c_dbl, _c_dbl, _c_dbl, _c_int, _c_int,
                       _c_dbl, _c_dbl, _c_int, _ptr, _ptr],
    "tk_forward_cone_3d": [_ptr, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl, _dptr, _dptr,
                           _c_int, _c_int, _c_int, _c_dbl, _ptr, _ptr],
    "tk_forward_cone_3d_bands": [_ptr, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl, _dptr, _dptr, _c_int,
                                 _c_int, _c_int, _c_dbl, _c_int, _c_int, ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.POINTER(_c_int), ctypes.POINTER(_c_int), _c_int, _ptr],
    "tk_forward_cone_3d_path": [_dptr, _dptr, _c_int, _c_int, _c_int, _c_int, _c_int, _c_int],
    "tk_fp_plan_create": [_ptr, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl,
                          ctypes.POINTER(ctypes.c_void_p), _ptr],
    "tk_fp_plan_project": [_ptr, _dptr, _dptr, _c_int, _c_int, _c_int, _c_dbl, _ptr, _ptr],
    "tk_fp_plan_destroy": [_ptr, _ptr],
    "tk_back_cone_3d": [_ptr, _c_int, _c_int, _c_int, _dptr, _c_dbl, _c_int, _c_int, _c_int, _c_int,
                        _c_dbl, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_back_cone_3d_ex": [_ptr, _c_int, _c_int, _c_int, _c_int, _c_int, _dptr, _c_dbl, _c_int,
                           _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl, _c_int, _c_int, _c_int,
                           _ptr, _ptr],
    "tk_forward_cone_3d_adjoint": [_ptr, _c_int, _c_int, _c_int, _dptr, _dptr, _c_int, _c_int,
                                   _c_int, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_forward_cone_3d_adjoint_ex": [_ptr, _c_int, _c_int, _c_int, _dptr, _dptr, _c_int, _c_int,
                                      _c_int, _c_dbl, _c_dbl, _c_dbl, _c_dbl, _c_int, _ptr, _ptr],
    "tk_back_cone_3d_adjoint": [_ptr, _c_int, _c_int, _c_int, _c_dbl, _c_dbl, _c_dbl, _dptr,
                                _c_dbl, _c_int, _c_int, _c_int, _c_int, _ptr, _ptr],
    "tk_forward_parallel_2d_adjoint": [_ptr, _c_int, _c_int, _dptr, _dptr, _c_dbl, _c_dbl, _c_int,
                                       _c_int, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_forward_fan_2d_adjoint": [_ptr, _c_int, _c_int, _dptr, _dptr, _c_dbl, _c_dbl, _c_dbl,
                                  _c_dbl, _c_int, _c_int, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_back_parallel_2d_adjoint": [_ptr, _c_int, _c_int, _c_dbl, _c_dbl, _dptr, _dptr, _c_int, _c_int, _c_dbl,
                                    _ptr, _ptr],
    "tk_back_fan_2d_adjoint": [_ptr, _c_int, _c_int, _c_dbl, _c_dbl, _dptr, _dptr, _c_int, _c_dbl, _c_dbl, _c_int,
                               _c_dbl, _c_int, _ptr, _ptr],
    "tk_fft_filter_rows": [_ptr, _c_ll, _c_int, _c_int, _dptr, _c_int, _c_dbl, _c_dbl, _c_dbl,
                           _c_dbl, _ptr, _ptr],
    "tk_fft_filter_rows_ex": [_ptr, _c_ll, _c_int, _c_int, _c_int, _c_int, _dptr, _c_int, _c_dbl,
                              _c_dbl, _c_dbl, _c_dbl, _ptr, _ptr],
    "tk_scale": [_ptr, _c_ll, _c_dbl, _ptr, _ptr],
    # sinogram degradation simulators (artifacts.py)
    "tk_jitter_shifts": [ctypes.c_ulonglong, _c_int, _c_int, ctypes.POINTER(ctypes.c_int)],
    "tk_detector_jitter": [_ptr, _c_int, _c_int, _c_int, _c_int, _c_int, ctypes.c_ulonglong, _ptr, _ptr],
    "tk_poisson_noise": [_ptr, _c_int, _c_ll, _c_dbl, _c_int, ctypes.c_ulonglong, _ptr, _ptr],
    "tk_gaussian_noise": [_ptr, _c_int, _c_ll, _c_dbl, _c_dbl, ctypes.c_ulonglong, _ptr, _ptr],
    "tk_ring_artifact": [_ptr, _c_int, _c_int, _c_int, ctypes.POINTER(ctypes.c_int), _c_int, _c_int, _c_int,
                         _c_int, _c_dbl, _ptr, _ptr],
    "tk_gantry_blur": [_ptr, _c_int, _c_int, _c_int, _dptr, _c_int, _ptr, _ptr],
}

_lock = threading.Lock()
_lib = None


class TkError(RuntimeError):
    """A CUDA or argument error reported by libtkb200.so."""


def load(path: Path | str | None = None):
    """Load (building first if absent) and type the shared library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            from . import build as _build

            _build.build()
        lib = ctypes.CDLL(str(p))
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            if name == "tk_last_error":
                fn.restype = ctypes.c_char_p
            elif name in ("tk_launch_count", "tk_cached_bytes"):
                fn.restype = ctypes.c_ulonglong
            else:
                fn.restype = _c_int
        _lib = lib
        return lib


def require_cuda(t: torch.Tensor, what: str) -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2511_08427_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor")


def stream_ptr(device: torch.device | None = None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dev_ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def host_f64(a: np.ndarray):
    """Keep-alive pair (array, ctypes pointer) for a host float64 argument."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_dptr)


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.tk_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(f"{name}: {msg}")
        raise TkError(f"{name}: {msg}")


def launch_count() -> int:
    return int(load().tk_launch_count())


def version() -> int:
    return int(load().tk_version())
