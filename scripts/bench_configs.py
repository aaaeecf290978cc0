"""Timings of the non-headline BASELINE configs (cfg1-cfg3) on the GPU next to the
float64 C oracle on the host cores (test infrastructure; the oracle is only timed
here, never shipped).  GPU: CUDA events around each device-resident operator, best
of 3 after a warm-up; CPU: one call each.  Prints one JSON object.

    cfg1  parallel 256^2 @1 mm, 180 angles over pi, 367 px @1 mm: FP + FBP
    cfg2  fan 512^2 @1 mm, 360 angles over 2 pi, 768 px @1.6 mm: FP + BP (+ weighted)
    cfg3  cone 256^3 @1 mm, 360 views, 512^2 @1.2 mm: FP + FDK
"""

import json
import math
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as ora  # noqa: E402
import paper_2511_08427_b200 as tk  # noqa: E402


def gpu_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return round(best, 3)


def cpu_ms(fn):
    t = time.perf_counter()
    out = fn()
    return round((time.perf_counter() - t) * 1e3, 1), out


res = {"cpu_threads": ora.num_threads()}

# cfg1 -------------------------------------------------------------------------
ang = tk.circular_trajectory_2d(180, math.pi)
g1 = tk.GeometryParallel2D((256, 256), (1.0, 1.0), 367, 1.0, ang)
x1 = tk.phantoms.shepp_logan_2d((256, 256)).cpu().numpy().astype(np.float64)
v1 = tk.Volume(x1, (1.0, 1.0))
s1 = tk.forward_project(v1, g1).data
sino1 = tk.Sinogram(s1, (1.0,))
c_fp, want = cpu_ms(lambda: ora.forward_parallel_2d(x1, (1.0, 1.0), ang, 367, 1.0, 0.5))
c_fbp, want_fbp = cpu_ms(lambda: ora.fbp_parallel_2d(want, ang, 1.0, (256, 256), (1.0, 1.0), "shepp_logan"))
res["cfg1"] = {"gpu_fp_ms": gpu_ms(lambda: tk.forward_project(v1, g1)),
               "gpu_fbp_ms": gpu_ms(lambda: tk.fbp_parallel_2d(sino1, g1, "shepp_logan")),
               "cpu_fp_ms": c_fp, "cpu_fbp_ms": c_fbp,
               "rel_fp": ora.rel_l2(s1.cpu().numpy(), want),
               "rel_fbp": ora.rel_l2(tk.fbp_parallel_2d(tk.Sinogram(want, (1.0,)), g1, "shepp_logan").data.cpu().numpy(),
                                     want_fbp)}

# cfg2 -------------------------------------------------------------------------
ang2 = tk.circular_trajectory_2d(360, 2 * math.pi)
g2 = tk.GeometryFan2D((512, 512), (1.0, 1.0), 768, 1.6, ang2, sdd=1200.0, sid=750.0)
x2 = tk.phantoms.shepp_logan_2d((512, 512)).cpu().numpy().astype(np.float64)
v2 = tk.Volume(x2, (1.0, 1.0))
s2 = tk.forward_project(v2, g2).data
sino2 = tk.Sinogram(s2, (1.6,))
c_fp2, want2 = cpu_ms(lambda: ora.forward_fan_2d(x2, (1.0, 1.0), ang2, 1200.0, 750.0, 768, 1.6, 0.5))
c_bp2, want_bp2 = cpu_ms(lambda: ora.back_fan_2d(want2, ang2, 1200.0, 750.0, 1.6, (512, 512), (1.0, 1.0), False))
res["cfg2"] = {"gpu_fp_ms": gpu_ms(lambda: tk.forward_project(v2, g2)),
               "gpu_bp_ms": gpu_ms(lambda: tk.back_project(sino2, g2)),
               "gpu_bp_weighted_ms": gpu_ms(lambda: tk.back_project(sino2, g2, fdk_weighting=True)),
               "cpu_fp_ms": c_fp2, "cpu_bp_ms": c_bp2,
               "rel_fp": ora.rel_l2(s2.cpu().numpy(), want2),
               "rel_bp": ora.rel_l2(tk.back_project(tk.Sinogram(want2, (1.6,)), g2).data.cpu().numpy(), want_bp2)}

# cfg3 -------------------------------------------------------------------------
g3 = tk.circular_cone_geometry((256,) * 3, (1.0,) * 3, (512, 512), (1.2, 1.2), 360, 2 * math.pi, 1200.0, 750.0)
x3 = tk.phantoms.shepp_logan_3d((256,) * 3)
v3 = tk.Volume(x3, (1.0,) * 3)
s3 = tk.forward_project(v3, g3).data
sino3 = tk.Sinogram(s3, (1.2, 1.2))
sub = g3.matrix_array()[::30]  # 12 views for the CPU sample (per-view cost is constant on a circle)
x3h = x3.cpu().numpy().astype(np.float64)
c_fp3, want3 = cpu_ms(lambda: ora.forward_cone_3d(x3h, (1.0,) * 3, sub, (512, 512), 0.5))
c_fdk3, _ = cpu_ms(lambda: ora.fdk_cone_3d(want3, sub, 1200.0, 750.0, (1.2, 1.2), (256,) * 3, (1.0,) * 3,
                                           "shepp_logan"))
res["cfg3"] = {"gpu_fp_ms": gpu_ms(lambda: tk.forward_project(v3, g3)),
               "gpu_fdk_ms": gpu_ms(lambda: tk.fdk_cone_3d(sino3, g3, "shepp_logan")),
               "cpu_fp_ms_extrapolated": round(c_fp3 * 30, 1), "cpu_fdk_ms_extrapolated": round(c_fdk3 * 30, 1),
               "cpu_sample": "12 of 360 views x 30",
               "rel_fp_12views": ora.rel_l2(s3[::30].cpu().numpy(), want3),
               "gups_fp": round(256**3 * 360 / (gpu_ms(lambda: tk.forward_project(v3, g3)) * 1e-3) / 1e9, 1)}
print(json.dumps(res))
