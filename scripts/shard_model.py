"""Per-rank compute of the multi-GPU decompositions, measured on ONE GPU.

For N in 1, 2, 4, 8 every rank's share of the cfg4 step is run and timed on the same
device, one rank after another (CUDA events):
  * forward projection of the rank's view block (coefficient cells built per rank);
  * z-slab FDK: filter of the rank's detector row band (all views) + back projection
    of its slab (the primary decomposition: disjoint slabs, no reduction);
  * angle-sharded FDK (comparison): filter + back projection of the rank's view block
    into a full partial volume, to be summed by a reduce / reduce-scatter.
The collectives themselves (sinogram all-gather, volume reduce) are NOT measured here
(no multi-GPU box); their bytes per rank are printed so the NVLink time can be added.
Prints one JSON object."""

import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import distributed as D  # noqa: E402
from paper_2511_08427_b200.filters import filter_stage_tensor  # noqa: E402
from paper_2511_08427_b200.projectors import bp_cone_tensor_ex, fp_tensor  # noqa: E402

VOL, VIEWS, DET = (512, 512, 512), 720, (1024, 1024)
geom = tk.circular_cone_geometry(VOL, (0.5,) * 3, DET, (0.6, 0.6), VIEWS, 2 * math.pi, 1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(VOL)
sino = fp_tensor(vol, geom, 0.25)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = ev(), ev()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


res = {}
for world in (1, 2, 4, 8):
    ranks = []
    for rank in range(world):
        vb, ve = D.shard_bounds(VIEWS, world, rank)
        sub = D.subset_geometry(geom, slice(vb, ve))
        z0, z1 = D.shard_bounds(VOL[0], world, rank)
        r0, r1 = D.row_band(geom, z0, z1) if world > 1 else (0, DET[0])
        loc = torch.empty((ve - vb, *DET), device="cuda")
        band_in = sino[:, r0:r1, :].contiguous()
        band = torch.empty_like(band_in)
        slab = torch.empty((z1 - z0, *VOL[1:]), device="cuda")
        part = torch.empty(VOL, device="cuda")
        filt_loc = torch.empty_like(loc)
        t_fp = timed(lambda: fp_tensor(vol, sub, 0.25, out=loc))
        t_zs = timed(lambda: (filter_stage_tensor(band_in, geom, "shepp_logan", out=band, row_offset=r0),
                              bp_cone_tensor_ex(band, geom, True, r0, z0, z1 - z0, out=slab)))
        t_as = timed(lambda: (filter_stage_tensor(sino[vb:ve], sub, "shepp_logan", out=filt_loc),
                              bp_cone_tensor_ex(filt_loc, sub, True, 0, 0, VOL[0], out=part)))
        ranks.append({"rank": rank, "views": ve - vb, "z": [z0, z1], "rows": [r0, r1],
                      "fp_ms": round(t_fp, 2), "fdk_zslab_ms": round(t_zs, 2), "fdk_angle_ms": round(t_as, 2)})
        del loc, band_in, band, slab, part, filt_loc
    gather_bytes = (world - 1) / world * VIEWS * DET[0] * DET[1] * 4 if world > 1 else 0
    reduce_bytes = (world - 1) / world * VOL[0] * VOL[1] * VOL[2] * 4 if world > 1 else 0
    res[world] = {
        "max_fp_ms": max(r["fp_ms"] for r in ranks),
        "max_fdk_zslab_ms": max(r["fdk_zslab_ms"] for r in ranks),
        "max_fdk_angle_ms": max(r["fdk_angle_ms"] for r in ranks),
        "allgather_recv_bytes_per_rank": int(gather_bytes),
        "reduce_bytes_per_rank": int(reduce_bytes),
        "ranks": ranks,
    }
print(json.dumps(res))
