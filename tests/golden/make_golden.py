"""Generate the golden fixtures in tests/golden/ by importing the REFERENCE itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

The reference (tomokit, /root/reference/pkg/src) is imported read-only; its
outputs on small seeded cases are stored as float64 .npz files next to this
script.  These fixtures pin the CPU oracle (oracle/) and, transitively, the
CUDA path.  Nothing on the GPU box reads /root/reference: only these committed
fixtures travel.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("TK_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import tomokit as tk  # noqa: E402
from tomokit import filters as tkf  # noqa: E402
from tomokit import projectors as tkp  # noqa: E402

OUT = Path(__file__).resolve().parent
SEED = 20240917


def save(name: str, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz: " + ", ".join(f"{k}{np.shape(v)}" for k, v in arrays.items()))


def main():
    rng = np.random.default_rng(SEED)

    # -- geometry ------------------------------------------------------------
    g = tk.circular_cone_geometry((16, 16, 16), (1.0, 1.0, 1.0), (12, 12), (1.6, 1.6), 8,
                                  2 * np.pi, 1200.0, 750.0)
    mats = g.matrix_array()
    _, sources, minv = tkp._cone_rays(g)
    g4 = tk.circular_cone_geometry((512, 512, 512), (0.5, 0.5, 0.5), (1024, 1024), (0.6, 0.6),
                                   720, 2 * np.pi, 1200.0, 750.0)
    mats4 = g4.matrix_array()
    # helical + sinusoidal poses (trajectory_from_poses), non-square detector
    thetas = np.linspace(0, 4 * np.pi, 10, endpoint=False)
    poses = []
    for th in thetas:
        zc = -6.0 + 12.0 * th / (4 * np.pi)
        ct, st = np.cos(th), np.sin(th)
        poses.append(tk.Pose(np.array([750.0 * ct, 750.0 * st, zc]),
                             np.array([-450.0 * ct, -450.0 * st, zc]),
                             np.array([-st, ct, 0.0]), np.array([0.0, 0.0, 1.0])))
    mats_helix = np.stack([m.entries for m in tk.trajectory_from_poses(poses, (10, 14), (1.5, 1.8))])
    sin_poses = []
    for th in np.linspace(0, 2 * np.pi, 9, endpoint=False):
        zc = 4.0 * np.sin(2 * th)
        ct, st = np.cos(th), np.sin(th)
        sin_poses.append(tk.Pose(np.array([750.0 * ct, 750.0 * st, zc]),
                                 np.array([-450.0 * ct, -450.0 * st, zc]),
                                 np.array([-st, ct, 0.0]), np.array([0.0, 0.0, 1.0])))
    mats_sin = np.stack([m.entries for m in tk.trajectory_from_poses(sin_poses, (12, 12), (1.6, 1.6))])
    # a tilted detector (u not horizontal) -- exercises the general (z-varying) path
    tilt = []
    for th in np.linspace(0, 2 * np.pi, 6, endpoint=False):
        ct, st = np.cos(th), np.sin(th)
        a = 0.2
        u = np.array([-st * np.cos(a), ct * np.cos(a), np.sin(a)])
        n = np.array([-ct, -st, 0.0])
        v = np.cross(n, u)
        v /= np.linalg.norm(v)
        tilt.append(tk.Pose(np.array([750.0 * ct, 750.0 * st, 0.0]),
                            np.array([-450.0 * ct, -450.0 * st, 0.0]), u, v))
    mats_tilt = np.stack([m.entries for m in tk.trajectory_from_poses(tilt, (12, 12), (1.6, 1.6))])
    raw = mats[3] * -2.5
    from_raw = tk.ProjectionMatrix.from_raw(raw).entries
    save("geometry", mats=mats, sources=sources, minv=minv, mats4=mats4, mats_helix=mats_helix,
         mats_sin=mats_sin, mats_tilt=mats_tilt, raw=raw, from_raw=from_raw,
         angles=tk.circular_trajectory_2d(24, 2 * np.pi))

    # -- parallel 2D ---------------------------------------------------------
    ang = tk.circular_trajectory_2d(24, 2 * np.pi)
    gp = tk.GeometryParallel2D((32, 32), (1.0, 1.0), 48, 1.0, ang)
    x = rng.standard_normal((32, 32))
    y = rng.standard_normal((24, 48))
    sl2 = tk.shepp_logan_2d((32, 32)).data
    gp2 = tk.GeometryParallel2D((20, 28), (0.7, 1.3), 37, 0.9, tk.circular_trajectory_2d(17, np.pi))
    x2 = rng.standard_normal((20, 28))
    y2 = rng.standard_normal((17, 37))
    save("parallel2d",
         x=x, y=y, angles=ang, fp=tkp.forward_project_parallel_2d(tk.Volume(x, (1.0, 1.0)), gp).data,
         fp_sl=tkp.forward_project_parallel_2d(tk.Volume(sl2, (1.0, 1.0)), gp).data, sl=sl2,
         bp=tkp.back_project_parallel_2d(tk.Sinogram(y, (1.0,)), gp).data,
         fp_step1=tkp.forward_project_parallel_2d(tk.Volume(x, (1.0, 1.0)), gp,
                                                  tkp.SamplingConfig(1.0)).data,
         x2=x2, y2=y2, angles2=gp2.angles,
         fp2=tkp.forward_project_parallel_2d(tk.Volume(x2, (0.7, 1.3)), gp2).data,
         bp2=tkp.back_project_parallel_2d(tk.Sinogram(y2, (0.9,)), gp2).data,
         fbp=tkf.fbp_parallel_2d(tk.Sinogram(y, (1.0,)), gp, "shepp_logan").data,
         fbp_ramp=tkf.fbp_parallel_2d(tk.Sinogram(y, (1.0,)), gp, "ramp").data)

    # -- fan 2D --------------------------------------------------------------
    gf = tk.GeometryFan2D((32, 32), (1.0, 1.0), 64, 1.6, ang, sdd=1200.0, sid=750.0)
    xf = rng.standard_normal((32, 32))
    yf = rng.standard_normal((24, 64))
    save("fan2d", x=xf, y=yf, angles=ang,
         fp=tkp.forward_project_fan_2d(tk.Volume(xf, (1.0, 1.0)), gf).data,
         bp=tkp.back_project_fan_2d(tk.Sinogram(yf, (1.6,)), gf, False).data,
         bpw=tkp.back_project_fan_2d(tk.Sinogram(yf, (1.6,)), gf, True).data,
         fbp=tkf.fbp_fan_2d(tk.Sinogram(yf, (1.6,)), gf, "cosine").data)

    # -- cone 3D -------------------------------------------------------------
    xc = rng.standard_normal((16, 16, 16))
    yc = rng.standard_normal((8, 12, 12))
    slc = tk.shepp_logan_3d((16, 16, 16)).data
    cfg = tkp.SamplingConfig(0.5)
    save("cone3d", x=xc, y=yc, sl=slc, mats=mats,
         fp=tkp.forward_project_cone_3d(tk.Volume(xc, (1.0, 1.0, 1.0)), g, cfg).data,
         fp_sl=tkp.forward_project_cone_3d(tk.Volume(slc, (1.0, 1.0, 1.0)), g, cfg).data,
         bp=tkp.back_project_cone_3d(tk.Sinogram(yc, (1.6, 1.6)), g, False).data,
         bpw=tkp.back_project_cone_3d(tk.Sinogram(yc, (1.6, 1.6)), g, True).data,
         filt=tkf.filter_stage(tk.Sinogram(yc, (1.6, 1.6)), g, "shepp_logan").data,
         fdk=tkf.fdk_cone_3d(tk.Sinogram(yc, (1.6, 1.6)), g, "shepp_logan").data)

    # anisotropic helical case: volume (14, 18, 16) @ (1.1, 0.9, 1.0), 10x14 detector
    gh = tk.GeometryCone3D((14, 18, 16), (1.1, 0.9, 1.0), (10, 14), (1.5, 1.8),
                           [tk.ProjectionMatrix(m) for m in mats_helix], 1200.0, 750.0)
    xh = rng.standard_normal((14, 18, 16))
    yh = rng.standard_normal((10, 10, 14))
    gt = tk.GeometryCone3D((12, 12, 12), (1.0, 1.0, 1.0), (12, 12), (1.6, 1.6),
                           [tk.ProjectionMatrix(m) for m in mats_tilt], 1200.0, 750.0)
    xt = rng.standard_normal((12, 12, 12))
    yt = rng.standard_normal((6, 12, 12))
    save("cone3d_general", xh=xh, yh=yh, mats_helix=mats_helix,
         fp_h=tkp.forward_project_cone_3d(tk.Volume(xh, (1.1, 0.9, 1.0)), gh, cfg).data,
         bp_h=tkp.back_project_cone_3d(tk.Sinogram(yh, (1.5, 1.8)), gh, True).data,
         xt=xt, yt=yt, mats_tilt=mats_tilt,
         fp_t=tkp.forward_project_cone_3d(tk.Volume(xt, (1.0, 1.0, 1.0)), gt, cfg).data,
         bp_t=tkp.back_project_cone_3d(tk.Sinogram(yt, (1.6, 1.6)), gt, True).data)

    # -- filters -------------------------------------------------------------
    w = {}
    for kind, make in (("ramp", tkf.ramp_filter), ("shepp_logan", tkf.shepp_logan_filter),
                       ("cosine", tkf.cosine_filter)):
        for width, sp in ((12, 1.0), (48, 0.625), (100, 1.3), (1024, 0.375)):
            w[f"{kind}_{width}"] = make(width, sp).weights
    rows = rng.standard_normal((3, 48))
    w["rows"] = rows
    w["rows_filtered"] = tkf.fft_filter(tk.Sinogram(rows, (1.0,)), tkf.shepp_logan_filter(48, 0.625)).data
    save("filters", **w)

    # -- tiny dense operators (exact A) for the transpose oracles -------------
    gpt = tk.GeometryParallel2D((5, 6), (1.0, 1.0), 9, 1.0, tk.circular_trajectory_2d(3, np.pi))
    gct = tk.circular_cone_geometry((4, 5, 6), (1.0, 1.0, 1.0), (5, 6), (1.6, 1.6), 3, 2 * np.pi,
                                    1200.0, 750.0)
    save("dense", A_par=tkp.materialize_operator(gpt, cfg, "forward"),
         B_par=tkp.materialize_operator(gpt, cfg, "back"),
         A_cone=tkp.materialize_operator(gct, cfg, "forward"),
         B_cone=tkp.materialize_operator(gct, cfg, "back"),
         ang_par=gpt.angles, mats_cone=gct.matrix_array())

    meta = {"seed": SEED, "reference": str(REF), "tomokit_version": tk.__version__,
            "numpy": np.__version__}
    (OUT / "golden_meta.json").write_text(json.dumps(meta, indent=2) + "\n")


if __name__ == "__main__":
    main()
