"""Forward-projection sample rate by detector row band (cfg4 geometry, 72 views):
rays of the central rows enter through an x / y face of the volume box, the top and
bottom rows' rays through a z face (their x/y cell crossings are not synchronised
within a quarter-warp).  Prints G samples/s per band."""

import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import fp_tensor  # noqa: E402

vol = tk.phantoms.shepp_logan_3d((512,) * 3)
res = {}
for rows, label in ((1024, "all rows"), (512, "central 512 rows"), (256, "central 256 rows")):
    g = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (rows, 1024), (0.6, 0.6), 720, 2 * math.pi,
                                  1200.0, 750.0)
    g = tk.GeometryCone3D(g.volume_shape, g.volume_spacing, g.detector_shape, g.detector_spacing,
                          g.matrices[::10], 1200.0, 750.0)
    out = torch.empty(g.sinogram_shape, device="cuda")
    fp_tensor(vol, g, 0.25, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        a.record()
        fp_tensor(vol, g, 0.25, out=out)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    n = bench.count_samples(g, 0.25, torch)
    res[label] = {"ms": round(best, 3), "samples": n, "gsamples_per_s": round(n / best / 1e6, 1)}
print(json.dumps(res))
