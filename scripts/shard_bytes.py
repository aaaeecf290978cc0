#!/usr/bin/env python3
"""Bytes each rank receives per cfg4 step under the three multi-GPU data paths
(host-only arithmetic over distributed.py's decomposition; no GPU):

  zslab     view-sharded FP -> uneven all-to-all of detector row bands -> z-slab FDK (default)
  gather    view-sharded FP -> all-gather of the whole sinogram -> z-slab FDK on the crop
  angle     view-sharded FP and FDK of the rank's own views -> reduce-scatter of partial volumes

    python scripts/shard_bytes.py [--out profiles/r02/shard_bytes.json]
"""
import argparse
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import distributed as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
a = ap.parse_args()
geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
V, (R, C) = geom.n_projections, geom.detector_shape
nz, ny, nx = geom.volume_shape
res = {}
for world in (1, 2, 4, 8):
    bands = D.slab_bands(geom, world)
    counts = [D.shard_bounds(V, world, g)[1] - D.shard_bounds(V, world, g)[0] for g in range(world)]
    rows = [r1 - r0 for (_, _, r0, r1) in bands]
    # all-to-all: rank h receives its band rows of every OTHER rank's views
    a2a = [4 * C * rows[h] * (V - counts[h]) for h in range(world)]
    gather = [4 * C * R * (V - counts[h]) for h in range(world)]
    # reduce-scatter of a (nz, ny, nx) fp32 partial: each rank receives (world-1)/world of a slab's worth x world
    rs = [4 * nx * ny * nz * (world - 1) // world if world > 1 else 0 for _ in range(world)]
    res[world] = {"band_rows": rows, "views_per_rank": counts,
                  "zslab_all_to_all_recv_GB_max": round(max(a2a) / 1e9, 3),
                  "all_gather_recv_GB_max": round(max(gather) / 1e9, 3),
                  "angle_reduce_scatter_recv_GB": round(max(rs) / 1e9, 3)}
    print(world, json.dumps(res[world]))
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
