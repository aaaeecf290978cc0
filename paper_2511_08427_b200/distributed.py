"""Multi-GPU decomposition of the cone-beam operators (one process per GPU).

Work is split only where it splits naturally (no reference counterpart; the
reference is single-process):

* forward projection -- contiguous view blocks per rank, volume replicated,
  no communication until the sinogram is exchanged (NCCL over NVLink): either
  one all-gather of the whole sinogram (`gather_views`), or -- what the FDK
  needs -- an uneven all-to-all that sends every rank only the detector row
  band of each view its z-slab projects into (`exchange_row_bands`), issued
  per view chunk so chunk k travels while chunk k+1 is projected
  (`forward_project_and_exchange`);
* FDK back projection -- z-slabs per rank; each rank filters and back-projects
  only the detector row band its slab projects into (band from the slab's
  corner projections through every P), so output slabs are disjoint and need
  no reduction;
* fused path (`forward_project_p2p`) -- the forward projection kernel itself
  stores each ray into the band buffers of the ranks whose z-slab needs its row,
  through peer (NVLink) addresses of symmetric-memory buffers: no separate
  collective, the exchange overlaps the projection ray by ray;
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
    "slab_bands",
    "chunk_bounds",
    "received_view_order",
    "exchange_row_bands",
    "forward_project_and_exchange",
    "forward_project_p2p",
    "fdk_angle_sharded",
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


# ---------------------------------------------------------------------------
# Row-band all-to-all (z-slab FDK fed by a view-sharded FP)
# ---------------------------------------------------------------------------


def slab_bands(geom: GeometryCone3D, world: int) -> list[tuple[int, int, int, int]]:
    """(z_begin, z_end, row_begin, row_end) of every rank's z-slab and detector row band."""
    out = []
    for r in range(world):
        z0, z1 = shard_bounds(geom.volume_shape[0], world, r)
        r0, r1 = row_band(geom, z0, z1) if world > 1 else (0, geom.detector_shape[0])
        out.append((z0, z1, r0, r1))
    return out


def chunk_bounds(n_views: int, n_chunks: int) -> list[tuple[int, int]]:
    """Local [begin, end) view offsets of each pipeline chunk (balanced, possibly empty)."""
    return [shard_bounds(n_views, n_chunks, k) for k in range(n_chunks)]


def received_view_order(n_views: int, world: int, n_chunks: int) -> np.ndarray:
    """Global view index of every view in the received band, in arrival layout:
    chunk-major, then source rank, then view.  The back projection takes the
    projection matrices in this order (its sum over views is order-free up to
    fp32 rounding), so the received band is used in place, without a reorder."""
    order = []
    starts = [shard_bounds(n_views, world, g)[0] for g in range(world)]
    counts = [shard_bounds(n_views, world, g)[1] - starts[g] for g in range(world)]
    for k in range(n_chunks):
        for g in range(world):
            b, e = shard_bounds(counts[g], n_chunks, k)
            order.extend(range(starts[g] + b, starts[g] + e))
    return np.asarray(order, dtype=np.int64)


def _all_to_all(out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits, group=None,
                async_op: bool = False):
    """all_to_all_single of 1-D tensors with uneven splits.  NCCL runs it on its
    own stream (async_op: returns the work handle); gloo on CUDA tensors is
    staged through host memory (functional path for the single-GPU check)."""
    if _backend() == "gloo" and inp.is_cuda:
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(o)
        return None
    return dist.all_to_all_single(out, inp, out_splits, in_splits, group=group, async_op=async_op)


def exchange_row_bands(local: torch.Tensor, counts: list[int], bands, rank: int, out: torch.Tensor,
                       group=None, async_op: bool = False):
    """Send rows [r0_h, r1_h) of this rank's views to every rank h; receive this
    rank's rows from every rank into ``out`` (sum(counts), r1 - r0, cols),
    source blocks in rank order.

    ``counts[g]`` = views rank g contributes in this exchange; ``bands[h]`` =
    (z0, z1, r0, r1) of rank h.  Bytes received per rank = 4 * cols * (r1 - r0)
    * sum(counts) -- its own band only, instead of the whole sinogram an
    all-gather delivers.  Returns (work or None, send buffer to keep alive).
    """
    v, rows, cols = local.shape
    if v != counts[rank]:
        raise ValueError("local view block does not match counts[rank]")
    my_rows = bands[rank][3] - bands[rank][2]
    if tuple(out.shape) != (sum(counts), my_rows, cols):
        raise ValueError("receive buffer does not match the band")
    parts = [local[:, r0:r1, :].reshape(-1) for (_, _, r0, r1) in bands]
    send = torch.cat(parts) if parts else local.new_empty(0)
    in_splits = [p.numel() for p in parts]
    out_splits = [c * my_rows * cols for c in counts]
    work = _all_to_all(out.view(-1), send, out_splits, in_splits, group=group, async_op=async_op)
    return work, send


def forward_project_and_exchange(vol: torch.Tensor, geom: GeometryCone3D, step: float, rank: int,
                                 world: int, n_chunks: int = 1, fp_fn: Callable | None = None,
                                 bands=None, out: torch.Tensor | None = None, group=None,
                                 on_chunk: Callable | None = None):
    """View-sharded forward projection whose output goes straight to the z-slab
    owners: chunk k of this rank's views is projected, then its row bands are
    sent with an asynchronous all-to-all while chunk k+1 is projected.

    Returns (band, order): band (V, r1 - r0, cols) holds this rank's detector
    rows of every view, in ``received_view_order`` layout; ``order`` are the
    global view indices of its rows.  ``on_chunk(k)`` is called after chunk k's
    projection is enqueued (timing hooks).
    """
    if fp_fn is None:
        from .projectors import fp_tensor as fp_fn
    nv = geom.n_projections
    bands = bands or slab_bands(geom, world)
    starts = [shard_bounds(nv, world, g)[0] for g in range(world)]
    counts = [shard_bounds(nv, world, g)[1] - starts[g] for g in range(world)]
    _, _, r0, r1 = bands[rank]
    rows, cols = geom.detector_shape
    if out is None:
        out = vol.new_empty((nv, r1 - r0, cols))
    pending, off = [], 0
    vb = starts[rank]
    for k in range(n_chunks):
        ck = [shard_bounds(counts[g], n_chunks, k) for g in range(world)]
        ccounts = [e - b for b, e in ck]
        total = sum(ccounts)
        if total == 0:
            continue
        b, e = ck[rank]
        if e > b:
            local = fp_fn(vol, subset_geometry(geom, slice(vb + b, vb + e)), step)
        else:
            local = vol.new_empty((0, rows, cols))
        if on_chunk is not None:
            on_chunk(k)
        if world == 1:
            out[off:off + total].copy_(local[:, r0:r1, :])
        else:
            pending.append(exchange_row_bands(local, ccounts, bands, rank, out[off:off + total],
                                              group=group, async_op=True))
        off += total
    for work, _send in pending:
        if work is not None:
            work.wait()
    return out, received_view_order(nv, world, n_chunks)


_symm_cache: dict = {}


def _band_buffers(shape, device, group):
    """A symmetric-memory (peer-addressable) fp32 buffer of ``shape`` on every rank and the
    list of every rank's buffer address (torch.distributed._symmetric_memory, CUDA IPC over
    NVLink); cached per (shape, device, group) -- allocation and rendezvous are collective."""
    import torch.distributed._symmetric_memory as symm

    group = group or dist.group.WORLD
    key = (tuple(shape), device.index, id(group))
    hit = _symm_cache.get(key)
    if hit is None:
        buf = symm.empty(shape, dtype=torch.float32, device=device)
        hdl = symm.rendezvous(buf, group)
        hit = _symm_cache[key] = (buf, hdl, [int(p) for p in hdl.buffer_ptrs])
    return hit


def forward_project_p2p(vol: torch.Tensor, geom: GeometryCone3D, step: float, rank: int, world: int,
                        bands=None, group=None, fp_bands_fn: Callable | None = None):
    """View-sharded forward projection fused with the row-band exchange.

    Rank g projects its view block and the kernel stores every ray straight into the
    band buffer of each rank h whose row band [r0_h, r1_h) holds the ray's detector row
    -- a peer address on another GPU (symmetric memory over NVLink), so the exchange
    IS the projection's output stores and needs no collective; a device-side barrier
    then makes all peers' stores visible.  Views land at their global index (no
    reordering).  Returns this rank's band (V, r1 - r0, cols), a view of the
    (V, max band rows, cols) symmetric buffer.
    """
    if fp_bands_fn is None:
        from .projectors import fp_bands_tensor as fp_bands_fn
    nv = geom.n_projections
    bands = bands or slab_bands(geom, world)
    rows, cols = geom.detector_shape
    pitch = max(r1 - r0 for (_, _, r0, r1) in bands)
    buf, hdl, ptrs = _band_buffers((nv, pitch, cols), vol.device, group)
    vb, ve = shard_bounds(nv, world, rank)
    hdl.barrier()  # every rank is done reading its band from the previous call
    if ve > vb:
        fp_bands_fn(vol, subset_geometry(geom, slice(vb, ve)), step, vb, ptrs,
                    [(r0, r1) for (_, _, r0, r1) in bands], pitch)
    hdl.barrier()  # all peers' stores into this rank's band are visible
    _, _, r0, r1 = bands[rank]
    return buf[:, : r1 - r0]


def fdk_angle_sharded(sino_local: torch.Tensor, geom: GeometryCone3D, filter_kind: str, rank: int,
                      world: int, filter_fn: Callable | None = None, bp_fn: Callable | None = None,
                      group=None) -> tuple[int, torch.Tensor]:
    """Comparison FDK: filter and back-project this rank's own views (full
    detector) into a full partial volume, then reduce-scatter z-slabs.  No
    sinogram exchange; (world - 1) / world of the volume crosses NVLink.
    Returns (z_begin, slab) scaled by pi / V; needs nz divisible by world."""
    from .filters import filter_stage_tensor
    from .projectors import bp_cone_tensor_ex

    nz = geom.volume_shape[0]
    if nz % world:
        raise ValueError("angle-sharded FDK needs nz divisible by the world size")
    b, e = shard_bounds(geom.n_projections, world, rank)
    filter_fn = filter_fn or (lambda s: filter_stage_tensor(s, geom, filter_kind))
    bp_fn = bp_fn or (lambda f: bp_cone_tensor_ex(f, geom, True, 0, 0, nz, views=slice(b, e)))
    part = bp_fn(filter_fn(sino_local))
    if world == 1:
        return 0, part.mul_(math.pi / geom.n_projections)
    out = part.new_empty((nz // world, *geom.volume_shape[1:]))
    if _backend() == "nccl":
        dist.reduce_scatter_tensor(out, part, group=group)
    else:
        dist.all_reduce(part, group=group)
        out.copy_(part[rank * (nz // world):(rank + 1) * (nz // world)])
    return rank * (nz // world), out.mul_(math.pi / geom.n_projections)
