"""Multi-GPU decomposition of the cone-beam operators (one process per GPU).

Work is split only where it splits naturally (no reference counterpart; the
reference is single-process):

* forward projection -- contiguous view blocks per rank, volume replicated,
  no communication until one all-gather of the sinogram (NCCL over NVLink);
* FDK back projection -- z-slabs per rank; each rank filters and back-projects
  only the detector row band its slab projects into (band from the slab's
  corner projections through every P), so output slabs are disjoint and need
  no reduction;
* comparison path -- angle-sharded back projection into full partial volumes
  followed by a reduce / reduce-scatter of the volume.

The compute callables are injectable so the orchestration (shard bounds, row
bands, collectives) can be exercised with the gloo backend on CPU.
"""

from __future__ import annotations

import math
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .geometry import GeometryCone3D

__all__ = [
    "shard_bounds",
    "row_band",
    "gather_views",
    "forward_project_view_sharded",
    "fdk_zslab",
    "back_project_angle_sharded",
    "subset_geometry",
]


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous [begin, end) of n items for `rank` of `world`."""
    q, r = divmod(int(n), int(world))
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def row_band(geom: GeometryCone3D, z_begin: int, z_end: int, views: slice | None = None,
             margin: int = 1) -> tuple[int, int]:
    """Detector rows [r0, r1) that voxels with z index in [z_begin, z_end) touch.

    Central projection of the slab's voxel-centre box is the convex hull of its
    8 projected corners (all in front of the source), so min/max over corners
    bounds every voxel's row coordinate; bilinear taps add row floor(fr) + 1.
    """
    nz, ny, nx = geom.volume_shape
    sz, sy, sx = geom.volume_spacing
    mats = geom.matrix_array() if views is None else geom.matrix_array()[views]
    xs = np.array([-(nx - 1) / 2.0, (nx - 1) / 2.0]) * sx
    ys = np.array([-(ny - 1) / 2.0, (ny - 1) / 2.0]) * sy
    zs = (np.array([z_begin, z_end - 1], dtype=np.float64) - (nz - 1) / 2.0) * sz
    corners = np.array([[x, y, z, 1.0] for x in xs for y in ys for z in zs])  # (8, 4)
    hom = np.einsum("vij,cj->vci", mats, corners)  # (V, 8, 3)
    w = hom[..., 2]
    if np.any(w <= 1e-12):  # slab reaches behind a source: keep every row
        return 0, geom.detector_shape[0]
    fr = hom[..., 1] / w
    rows = geom.detector_shape[0]
    # taps touch rows floor(fr) and floor(fr) + 1; `margin` rows absorb fp32 rounding
    r0 = int(math.floor(float(fr.min()))) - margin
    r1 = int(math.floor(float(fr.max()))) + 2 + margin
    return max(0, min(rows, r0)), max(0, min(rows, r1))


def subset_geometry(geom: GeometryCone3D, views: slice) -> GeometryCone3D:
    """The same scan restricted to a block of views."""
    return GeometryCone3D(geom.volume_shape, geom.volume_spacing, geom.detector_shape,
                          geom.detector_spacing, geom.matrices[views], geom.sdd, geom.sid)


def _backend() -> str:
    return dist.get_backend() if dist.is_initialized() else "none"


def gather_views(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """All-gather per-rank view blocks (possibly uneven) into the full stack.

    NCCL: one all_gather_into_tensor over equal padded blocks; other backends:
    all_gather of a tensor list.
    """
    world = len(counts)
    if world == 1:
        return local
    vmax = max(counts)
    pad = local.new_zeros((vmax, *local.shape[1:]))
    pad[: local.shape[0]] = local
    if _backend() == "nccl":
        full = local.new_empty((world * vmax, *local.shape[1:]))
        dist.all_gather_into_tensor(full, pad, group=group)
        parts = [full[i * vmax: i * vmax + counts[i]] for i in range(world)]
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        parts = [bufs[i][: counts[i]] for i in range(world)]
    if all(c == vmax for c in counts) and _backend() == "nccl":
        return full
    return torch.cat(parts, dim=0)


def forward_project_view_sharded(vol: torch.Tensor, geom: GeometryCone3D, step: float,
                                 rank: int, world: int, fp_fn: Callable | None = None,
                                 gather: bool = True, group=None) -> torch.Tensor:
    """Rank-local views of A x, then (optionally) the all-gathered sinogram."""
    if fp_fn is None:
        from .projectors import fp_tensor as fp_fn
    counts = [shard_bounds(geom.n_projections, world, r)[1] - shard_bounds(geom.n_projections, world, r)[0]
              for r in range(world)]
    b, e = shard_bounds(geom.n_projections, world, rank)
    local = fp_fn(vol, subset_geometry(geom, slice(b, e)), step)
    return gather_views(local, counts, group) if gather else local


def fdk_zslab(sino: torch.Tensor, geom: GeometryCone3D, filter_kind: str, rank: int, world: int,
              filter_fn: Callable | None = None, bp_fn: Callable | None = None):
    """FDK of this rank's z-slab from the full sinogram, touching only its row band.

    Returns (z_begin, slab) with slab (z_count, ny, nx).
    """
    from .filters import filter_stage_tensor
    from .projectors import bp_cone_tensor_ex

    filter_fn = filter_fn or (lambda s, r0: filter_stage_tensor(s, geom, filter_kind, row_offset=r0))
    bp_fn = bp_fn or (lambda band, r0, z0, nzl: bp_cone_tensor_ex(band, geom, True, r0, z0, nzl))
    z0, z1 = shard_bounds(geom.volume_shape[0], world, rank)
    if z1 <= z0:
        return z0, sino.new_zeros((0, *geom.volume_shape[1:]))
    r0, r1 = row_band(geom, z0, z1)
    if r1 <= r0:
        return z0, sino.new_zeros((z1 - z0, *geom.volume_shape[1:]))
    # rows [r0, r1) of every view, filtered with their global row offset (the
    # cosine pre-weight depends on the detector v coordinate)
    band = filter_fn(sino[:, r0:r1, :].contiguous(), r0)
    slab = bp_fn(band, r0, z0, z1 - z0)
    slab.mul_(math.pi / geom.n_projections)
    return z0, slab


def back_project_angle_sharded(sino_local: torch.Tensor, geom: GeometryCone3D, weighted: bool,
                               rank: int, world: int, bp_fn: Callable | None = None,
                               op: str = "reduce", group=None) -> torch.Tensor:
    """Comparison path: back-project this rank's view block into a full partial
    volume, then reduce to rank 0 (op="reduce") or reduce-scatter z-slabs
    (op="reduce_scatter", equal slabs required)."""
    if bp_fn is None:
        from .projectors import bp_tensor as bp_fn
    b, e = shard_bounds(geom.n_projections, world, rank)
    part = bp_fn(sino_local, subset_geometry(geom, slice(b, e)), weighted)
    if world == 1:
        return part
    if op == "reduce":
        dist.reduce(part, dst=0, group=group)
        return part
    nz = geom.volume_shape[0]
    if nz % world:
        raise ValueError("reduce_scatter needs nz divisible by the world size")
    out = part.new_empty((nz // world, *geom.volume_shape[1:]))
    if _backend() == "nccl":
        dist.reduce_scatter_tensor(out, part, group=group)
    else:
        dist.all_reduce(part, group=group)
        out.copy_(part[rank * (nz // world):(rank + 1) * (nz // world)])
    return out
