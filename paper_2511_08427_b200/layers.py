"""PYRO-NN style differentiable operators (torch.autograd.Function + nn.Module).

Forward/back projector pairs for parallel 2D, fan 2D and cone 3D, on CUDA
tensors, with two adjoint conventions:

* ``adjoint="paired"`` (default, the reference's convention,
  /root/reference/pkg/src/tomokit/autodiff.py:1-19, 59-68): the gradient of
  the ray-driven projection A is the unweighted voxel-driven back projection B
  and vice versa.  Cheap, gather-only, deterministic -- but not an exact
  transpose (the reference's measured defect is 1e-3).
* ``adjoint="matched"``: exact transposes A^T / B^T (scatter kernels), so the
  dot-product test <Ax, y> = <x, A^T y> holds to fp32 round-off and the
  gradients are correctly scaled at any detector pitch.

Inputs may carry leading batch dimensions: (..., *volume_shape) projects each
item.  The reference's own torch layer (bindings/.../torch_layer.py:18-41)
copies to host numpy and back on every call; here everything stays on the GPU.
"""

from __future__ import annotations

import torch

from .geometry import GeometryCone3D, GeometryFan2D, GeometryParallel2D
from .projectors import SamplingConfig, bp_adjoint_tensor, bp_tensor, fp_adjoint_tensor, fp_tensor

__all__ = [
    "ParallelProjection2D",
    "ParallelBackProjection2D",
    "FanProjection2D",
    "FanBackProjection2D",
    "ConeProjection3D",
    "ConeBackProjection3D",
    "ParallelProjectionFor2D",
    "ParallelBackProjectionFor2D",
    "FanProjectionFor2D",
    "FanBackProjectionFor2D",
    "ConeProjectionFor3D",
    "ConeBackProjectionFor3D",
]

_ADJ = ("paired", "matched")


def _batched(fn, x: torch.Tensor, item_shape: tuple, out_shape: tuple) -> torch.Tensor:
    lead = tuple(x.shape[: x.dim() - len(item_shape)])
    if tuple(x.shape[len(lead):]) != tuple(item_shape):
        raise ValueError(f"expected trailing shape {tuple(item_shape)}, got {tuple(x.shape)}")
    if not lead:
        return fn(x)
    flat = x.reshape(-1, *item_shape)
    out = torch.empty((flat.shape[0], *out_shape), dtype=torch.float32, device=x.device)
    for i in range(flat.shape[0]):
        fn(flat[i], out[i])
    return out.reshape(*lead, *out_shape)


def _project(x, geom, step):
    return _batched(lambda v, o=None: fp_tensor(v, geom, step, out=o), x, geom.volume_shape,
                    geom.sinogram_shape)


def _backproject(y, geom, weighted):
    return _batched(lambda s, o=None: bp_tensor(s, geom, weighted, out=o), y, geom.sinogram_shape,
                    geom.volume_shape)


def _project_T(y, geom, step):
    def one(s, o=None):
        r = fp_adjoint_tensor(s, geom, step)
        if o is not None:
            o.copy_(r)
        return r

    return _batched(one, y, geom.sinogram_shape, geom.volume_shape)


def _backproject_T(x, geom, weighted):
    def one(v, o=None):
        r = bp_adjoint_tensor(v, geom, weighted)
        if o is not None:
            o.copy_(r)
        return r

    return _batched(one, x, geom.volume_shape, geom.sinogram_shape)


class _Projection(torch.autograd.Function):
    """y = A x (ray-driven).  backward: paired B, or exact A^T."""

    @staticmethod
    def forward(ctx, volume, geometry, adjoint="paired", sampling=None):
        if adjoint not in _ADJ:
            raise ValueError(f"adjoint must be one of {_ADJ}")
        cfg = sampling or SamplingConfig()
        step = cfg.step(geometry.volume_spacing)
        ctx.geometry, ctx.adjoint, ctx.step = geometry, adjoint, step
        return _project(volume.detach(), geometry, step)

    @staticmethod
    def backward(ctx, grad):
        grad = grad.contiguous().float()
        if ctx.adjoint == "matched":
            g = _project_T(grad, ctx.geometry, ctx.step)
        else:  # autodiff.py:59-62: unweighted paired back projection
            g = _backproject(grad, ctx.geometry, False)
        return g, None, None, None


class _BackProjection(torch.autograd.Function):
    """x = B y (voxel-driven, optionally (sid/w)^2 weighted).
    backward: paired A (unweighted only, autodiff.py:65-68), or exact B^T."""

    @staticmethod
    def forward(ctx, sinogram, geometry, adjoint="paired", fdk_weighting=False, sampling=None):
        if adjoint not in _ADJ:
            raise ValueError(f"adjoint must be one of {_ADJ}")
        if fdk_weighting and isinstance(geometry, GeometryParallel2D) and not isinstance(geometry, GeometryFan2D):
            raise ValueError("parallel backprojection has no distance weighting")
        cfg = sampling or SamplingConfig()
        ctx.geometry, ctx.adjoint, ctx.weighted = geometry, adjoint, bool(fdk_weighting)
        ctx.step = cfg.step(geometry.volume_spacing)
        return _backproject(sinogram.detach(), geometry, bool(fdk_weighting))

    @staticmethod
    def backward(ctx, grad):
        grad = grad.contiguous().float()
        if ctx.adjoint == "matched":
            g = _backproject_T(grad, ctx.geometry, ctx.weighted)
        else:
            if ctx.weighted:
                raise NotImplementedError("the paired adjoint excludes distance weighting "
                                          "(autodiff.py:10-11); use adjoint='matched'")
            g = _project(grad, ctx.geometry, ctx.step)
        return g, None, None, None, None


def _typed(kind):
    def check(geom):
        if not isinstance(geom, kind):
            raise TypeError(f"expected {kind.__name__}, got {type(geom).__name__}")
        return geom

    return check


class ParallelProjection2D(_Projection):
    @staticmethod
    def forward(ctx, volume, geometry, adjoint="paired", sampling=None):
        _typed(GeometryParallel2D)(geometry)
        return _Projection.forward(ctx, volume, geometry, adjoint, sampling)


class FanProjection2D(_Projection):
    @staticmethod
    def forward(ctx, volume, geometry, adjoint="paired", sampling=None):
        _typed(GeometryFan2D)(geometry)
        return _Projection.forward(ctx, volume, geometry, adjoint, sampling)


class ConeProjection3D(_Projection):
    @staticmethod
    def forward(ctx, volume, geometry, adjoint="paired", sampling=None):
        _typed(GeometryCone3D)(geometry)
        return _Projection.forward(ctx, volume, geometry, adjoint, sampling)


class ParallelBackProjection2D(_BackProjection):
    @staticmethod
    def forward(ctx, sinogram, geometry, adjoint="paired", fdk_weighting=False, sampling=None):
        _typed(GeometryParallel2D)(geometry)
        return _BackProjection.forward(ctx, sinogram, geometry, adjoint, fdk_weighting, sampling)


class FanBackProjection2D(_BackProjection):
    @staticmethod
    def forward(ctx, sinogram, geometry, adjoint="paired", fdk_weighting=False, sampling=None):
        _typed(GeometryFan2D)(geometry)
        return _BackProjection.forward(ctx, sinogram, geometry, adjoint, fdk_weighting, sampling)


class ConeBackProjection3D(_BackProjection):
    @staticmethod
    def forward(ctx, sinogram, geometry, adjoint="paired", fdk_weighting=False, sampling=None):
        _typed(GeometryCone3D)(geometry)
        return _BackProjection.forward(ctx, sinogram, geometry, adjoint, fdk_weighting, sampling)


class _Layer(torch.nn.Module):
    """PYRO-NN layer object: ``ConeProjectionFor3D().forward(x, geometry)``."""

    fn = None

    def __init__(self, adjoint: str = "paired", **kwargs):
        super().__init__()
        self.adjoint = adjoint
        self.kwargs = kwargs

    def forward(self, x, geometry):
        if hasattr(geometry, "build"):  # PYRO-NN Geometry front end
            geometry = geometry.build()
        x = torch.as_tensor(x)
        if not x.is_cuda:
            x = x.cuda()
        return type(self).fn.apply(x.float(), geometry, self.adjoint, *self.kwargs.values())


class ParallelProjectionFor2D(_Layer):
    fn = ParallelProjection2D


class FanProjectionFor2D(_Layer):
    fn = FanProjection2D


class ConeProjectionFor3D(_Layer):
    fn = ConeProjection3D


class _BackLayer(_Layer):
    def __init__(self, adjoint: str = "paired", fdk_weighting: bool = False):
        super().__init__(adjoint, fdk_weighting=fdk_weighting)


class ParallelBackProjectionFor2D(_BackLayer):
    fn = ParallelBackProjection2D


class FanBackProjectionFor2D(_BackLayer):
    fn = FanBackProjection2D


class ConeBackProjectionFor3D(_BackLayer):
    fn = ConeBackProjection3D
