"""Forward-projector throughput on the central detector rows only (whose rays
keep a thin z-slab of the volume L2-resident) vs the full detector: general
ray-per-thread kernel vs the z-mirror-pair kernel, cfg4 geometry otherwise.

    python scripts/fp_band_probe.py [--rows 64 128 1024]
"""
import argparse
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import fp_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, nargs="+", default=[32, 64, 128, 256, 1024])
ap.add_argument("--configs", default="TK_FP_MIRROR=0;TK_FP_MIRROR=1")
a = ap.parse_args()
vol = tk.phantoms.shepp_logan_3d((512,) * 3)
res = {}
for rows in a.rows:
    geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (rows, 1024), (0.6, 0.6), 720, 2 * math.pi,
                                     1200.0, 750.0)
    sino = torch.empty(geom.sinogram_shape, device="cuda")
    for cfg in a.configs.split(";"):
        os.environ.update(dict(kv.split("=") for kv in cfg.split(",") if kv))
        fp_tensor(vol, geom, 0.25, out=sino)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(3):
            s.record()
            fp_tensor(vol, geom, 0.25, out=sino)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        res[f"rows={rows} {cfg}"] = {"ms": round(best, 3), "ms_per_row": round(best / rows, 4)}
        print(f"rows={rows} {cfg}: {best:.3f} ms ({best / rows:.4f} ms/row)", flush=True)
print(json.dumps(res))
