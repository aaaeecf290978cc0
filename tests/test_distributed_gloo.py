"""Multi-rank orchestration on CPU (gloo, world_size 2): view-sharded forward
projection + all-gather, z-slab FDK with cropped row bands, angle-sharded back
projection + reduce.  The per-rank compute is the float64 oracle injected as
the kernel, so this exercises exactly the host logic the NCCL path runs."""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _geom():
    import paper_2511_08427_b200 as tk

    return tk.circular_cone_geometry((20, 18, 16), (1.0, 1.1, 0.9), (30, 28), (1.3, 1.3), 10, 2 * np.pi,
                                     1200.0, 750.0)


def _oracle_fns(geom):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as ora

    def fp_fn(vol, g, step):
        out = ora.forward_cone_3d(vol.double().numpy(), g.volume_spacing, g.matrix_array(), g.detector_shape, step)
        return torch.from_numpy(out).float()

    def filter_fn(band, r0):
        rows, cols = geom.detector_shape
        dv, du = geom.detector_spacing
        u = (np.arange(cols) - (cols - 1) / 2.0) * du
        v = (np.arange(r0, r0 + band.shape[1]) - (rows - 1) / 2.0) * dv
        w = geom.sdd / np.sqrt(geom.sdd**2 + u[None, :] ** 2 + v[:, None] ** 2)
        pitch = du * geom.sid / geom.sdd
        wts = ora.filter_weights("shepp_logan", cols, pitch)
        return torch.from_numpy(ora.fft_filter(band.double().numpy() * w, wts, pitch)).float()

    def bp_fn(band, r0, z0, nzl):
        full = np.zeros(geom.sinogram_shape)
        full[:, r0:r0 + band.shape[1]] = band.double().numpy()
        vol = ora.back_cone_3d(full, geom.matrix_array(), geom.sid, geom.volume_shape, geom.volume_spacing, True)
        return torch.from_numpy(vol[z0:z0 + nzl]).float()

    def bp_full(sino, g, weighted):
        return torch.from_numpy(ora.back_cone_3d(sino.double().numpy(), g.matrix_array(), g.sid, g.volume_shape,
                                                 g.volume_spacing, weighted)).float()

    return ora, fp_fn, filter_fn, bp_fn, bp_full


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2511_08427_b200 import distributed as D

        geom = _geom()
        ora, fp_fn, filter_fn, bp_fn, bp_full = _oracle_fns(geom)
        rng = np.random.default_rng(0)
        x = torch.from_numpy(rng.standard_normal(geom.volume_shape)).float()
        sino = D.forward_project_view_sharded(x, geom, 0.45, rank, world, fp_fn=fp_fn)
        z0, slab = D.fdk_zslab(sino, geom, "shepp_logan", rank, world, filter_fn=filter_fn, bp_fn=bp_fn)
        slabs = [None] * world
        dist.all_gather_object(slabs, (z0, slab.numpy()))
        vb, ve = D.shard_bounds(geom.n_projections, world, rank)
        part = D.back_project_angle_sharded(sino[vb:ve].contiguous(), geom, True, rank, world, bp_fn=bp_full)
        if rank == 0:
            q.put(("ok", sino.numpy(), slabs, part.numpy()))
    except Exception as exc:  # noqa: BLE001
        q.put(("err", repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_sharded_pipeline_matches_single_process():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as ora

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = mp.start_processes(_worker, args=(world, _free_port(), q), nprocs=world, join=False,
                               start_method="spawn")
    res = q.get()  # read before joining: the payload is larger than the pipe buffer
    while not procs.join():
        pass
    assert res[0] == "ok", res
    _, sino, slabs, part = res
    geom = _geom()
    x = np.random.default_rng(0).standard_normal(geom.volume_shape)
    mats = geom.matrix_array()
    want_sino = ora.forward_cone_3d(x, geom.volume_spacing, mats, geom.detector_shape, 0.45)
    np.testing.assert_allclose(sino, want_sino, rtol=0, atol=1e-5 * np.abs(want_sino).max())
    # z-slab FDK from cropped row bands == full-volume FDK
    want_fdk = ora.fdk_cone_3d(sino.astype(np.float64), mats, geom.sdd, geom.sid, geom.detector_spacing,
                               geom.volume_shape, geom.volume_spacing, "shepp_logan")
    got = np.concatenate([s for _, s in sorted(slabs, key=lambda t: t[0])], axis=0)
    assert got.shape == want_fdk.shape
    assert ora.rel_l2(got, want_fdk) < 1e-5
    # angle-sharded back projection + reduce == full back projection
    want_bp = ora.back_cone_3d(sino.astype(np.float64), mats, geom.sid, geom.volume_shape, geom.volume_spacing, True)
    assert ora.rel_l2(part, want_bp) < 1e-5
