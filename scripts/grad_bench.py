"""cfg5 timing: one gradient step of 0.5 ||A x - y||^2 through ConeProjection3D on a
helical (or sinusoidal) 512^3 / 720-view / 1024^2 trajectory, both adjoint conventions,
plus the bare matched-adjoint kernels (A^T y, B^T x)."""

import argparse
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import bp_adjoint_tensor, bp_tensor, fp_adjoint_tensor, fp_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--traj", default="helical")
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--views", type=int, default=720)
ap.add_argument("--det", type=int, default=1024)
a = ap.parse_args()

n, det = a.n, a.det
vs, ds = 256.0 / n, 614.4 / det
if a.traj == "helical":
    mats = tk.helical_trajectory_3d(a.views, 4 * math.pi, 1200.0, 750.0, (det, det), (ds, ds), -64.0, 64.0)
else:
    mats = tk.sinusoidal_trajectory_3d(a.views, 2 * math.pi, 1200.0, 750.0, (det, det), (ds, ds), 20.0)
geom = tk.GeometryCone3D((n,) * 3, (vs,) * 3, (det, det), (ds, ds), mats, 1200.0, 750.0)
x0 = tk.phantoms.shepp_logan_3d(geom.volume_shape)
y = fp_tensor(x0, geom, 0.5 * vs)
y += 0.01 * torch.randn_like(y)


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return round(best, 2)


res = {"traj": a.traj, "shape": [n, a.views, det]}
for adj in ("paired", "matched"):
    def step():
        x = x0.clone().requires_grad_(True)
        r = tk.ConeProjection3D.apply(x, geom, adj) - y
        loss = 0.5 * (r * r).sum()
        loss.backward()
        return x.grad
    res[f"grad_step_ms_{adj}"] = timed(step)
res["fp_ms"] = timed(lambda: fp_tensor(x0, geom, 0.5 * vs))
res["bp_ms"] = timed(lambda: bp_tensor(y, geom, False))
res["fp_adjoint_ms"] = timed(lambda: fp_adjoint_tensor(y, geom, 0.5 * vs))
res["fp_adjoint_deterministic_ms"] = timed(lambda: fp_adjoint_tensor(y, geom, 0.5 * vs, deterministic=True))
res["bp_adjoint_ms"] = timed(lambda: bp_adjoint_tensor(x0, geom, False))
print(json.dumps(res))
