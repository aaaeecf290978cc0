"""Forward-projection cost per view as a function of the view angle (cfg4 geometry).

Projects blocks of --block consecutive views (0.5 deg apart) starting at 0, 5, ..., 45 deg
through one ForwardProjectionPlan and prints ms per view for each block."""

import argparse
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import ForwardProjectionPlan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--block", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi,
                                 1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
out = torch.empty((a.block, 1024, 1024), device="cuda")
res = {}
with ForwardProjectionPlan(vol, geom) as plan:
    for deg in range(0, 50, 5):
        i0 = deg * 2
        views = slice(i0, i0 + a.block)
        plan.project(views, out, 0.25)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(a.reps):
            s.record()
            plan.project(views, out, 0.25)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        res[deg] = round(best / a.block, 4)
print(json.dumps({"ms_per_view_by_angle_deg": res}))
