"""Measurements of the SURVEY §8(f) "next" rows built around the hot path, GPU against the
unmodified reference (tomokit from baseline/_ref) on the host:

  artifacts   detector jitter, Poisson (transmission), Gaussian, ring, gantry blur on a cfg4-sized
              sinogram (720 x 1024 x 1024); the reference on a 24-view slice (its cost is linear in
              views), GPU on all 720 views -- reported per view
  grid I/O    write_grid + read_grid of a 512^3 volume (f32le .raw + .json), both implementations,
              through /tmp
  geometry    helical 720-view trajectory from poses + the per-view ray constants the forward
              projector needs (reference: projectors._cone_rays)

    python scripts/bench_next.py [--out profiles/r02/bench_next.json]
"""
import argparse
import json
import math
import os
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="")
a = ap.parse_args()

ref = None
if (ROOT / "baseline" / "_ref" / "tomokit").is_dir():
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tk_numba_cache")
    import tomokit as ref  # noqa: E402


def gpu_ms(fn, reps=3):
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
    return best


def cpu_ms(fn, reps=1):
    fn()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


V, R, C, SUB = 720, 1024, 1024, 24
res = {"artifacts": {}, "grid_io": {}, "geometry": {}}
geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (R, C), (0.6, 0.6), V, 2 * math.pi, 1200.0, 750.0)
sino = tk.Sinogram(torch.rand(V, R, C, device="cuda") * 2.0, (0.6, 0.6))
ops = {
    "jitter": lambda m, s: m.add_detector_jitter(s, 3, "u", seed=1),
    "poisson": lambda m, s: m.add_poisson_noise(s, 1e5, "transmission", seed=2),
    "gaussian": lambda m, s: m.add_gaussian_noise(s, 0.0, 0.05, seed=3),
    "ring": lambda m, s: m.add_ring_artifact(s, [100, 500, 900], (0, s.data.shape[0]), mode="zero"),
}
rsub = None
if ref is not None:
    rsub = ref.Sinogram(np.random.default_rng(0).uniform(0, 2, (SUB, R, C)), (0.6, 0.6))
    rgeom = ref.GeometryCone3D((512,) * 3, (0.5,) * 3, (R, C), (0.6, 0.6),
                               ref.circular_trajectory_3d(V, 2 * math.pi, 1200.0, 750.0, (R, C), (0.6, 0.6))[:SUB],
                               1200.0, 750.0)
for name, op in ops.items():
    g = gpu_ms(lambda: op(tk, sino))
    row = {"gpu_ms_720_views": round(g, 3), "gpu_ms_per_view": round(g / V, 5)}
    if ref is not None:
        c = cpu_ms(lambda: op(ref, rsub))
        row.update({"ref_cpu_ms_24_views": round(c, 1), "ref_cpu_ms_per_view": round(c / SUB, 3),
                    "speedup_per_view": round((c / SUB) / (g / V), 1)})
    res["artifacts"][name] = row
    print(name, row, flush=True)
g = gpu_ms(lambda: tk.add_gantry_motion_blur(sino, geom, 5))
row = {"gpu_ms_720_views": round(g, 3), "gpu_ms_per_view": round(g / V, 5)}
if ref is not None:
    c = cpu_ms(lambda: ref.add_gantry_motion_blur(rsub, rgeom, 5))
    row.update({"ref_cpu_ms_24_views": round(c, 1), "ref_cpu_ms_per_view": round(c / SUB, 3),
                "speedup_per_view": round((c / SUB) / (g / V), 1)})
res["artifacts"]["gantry_blur"] = row
print("gantry_blur", row, flush=True)

vol = tk.Volume(torch.rand(512, 512, 512, device="cuda"), (0.5,) * 3)
with tempfile.TemporaryDirectory() as d:
    p = Path(d) / "vol"
    w = cpu_ms(lambda: tk.write_grid(vol, p), reps=2)
    r = cpu_ms(lambda: tk.read_grid(p), reps=2)
    res["grid_io"]["ours_write_ms"], res["grid_io"]["ours_read_to_device_ms"] = round(w, 1), round(r, 1)
    if ref is not None:
        rv = ref.Volume(np.random.default_rng(1).uniform(0, 1, (512, 512, 512)), (0.5,) * 3)
        q = Path(d) / "rvol"
        res["grid_io"]["ref_write_ms"] = round(cpu_ms(lambda: ref.write_grid(rv, q), reps=2), 1)
        res["grid_io"]["ref_read_ms"] = round(cpu_ms(lambda: ref.read_grid(q), reps=2), 1)
print("grid_io", res["grid_io"], flush=True)


def ours_geom():
    mats = tk.helical_trajectory_3d(V, 4 * math.pi, 1200.0, 750.0, (R, C), (0.6, 0.6), -64.0, 64.0)
    gg = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (R, C), (0.6, 0.6), mats, 1200.0, 750.0)
    return gg.ray_constants


res["geometry"]["ours_helical_720_ms"] = round(cpu_ms(ours_geom, reps=3), 2)
if ref is not None:
    from tomokit import projectors as rp

    th = np.arange(V) * 4 * math.pi / V
    z = -64.0 + 128.0 * th / (4 * math.pi)

    def ref_geom():
        poses = [ref.Pose(np.array([750 * math.cos(t), 750 * math.sin(t), zz]),
                          np.array([-450 * math.cos(t), -450 * math.sin(t), zz]),
                          np.array([-math.sin(t), math.cos(t), 0.0]), np.array([0.0, 0.0, 1.0]))
                 for t, zz in zip(th, z)]
        mats = ref.trajectory_from_poses(poses, (R, C), (0.6, 0.6))
        gg = ref.GeometryCone3D((512,) * 3, (0.5,) * 3, (R, C), (0.6, 0.6), mats, 1200.0, 750.0)
        return rp._cone_rays(gg)

    try:
        res["geometry"]["ref_helical_720_ms"] = round(cpu_ms(ref_geom, reps=3), 2)
    except Exception as exc:  # noqa: BLE001
        res["geometry"]["ref_error"] = repr(exc)[:200]
print("geometry", res["geometry"], flush=True)
print(json.dumps(res))
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
