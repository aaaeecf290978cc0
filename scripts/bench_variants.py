"""Time the forward / back projector kernel variants at cfg4 -- the default kernels
against the measured comparisons the north star asks for (texture unit, the
warp-cooperative march, the general-P quad back projector) -- and report each
result's relative L2 difference from the first one listed.

    python scripts/bench_variants.py [--views 720] [--reps 3] [--out gpurun_out/variants.json]
"""

import argparse
import json
import math
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.filters import filter_stage_tensor  # noqa: E402
from paper_2511_08427_b200.projectors import bp_tensor, fp_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=720)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--fp", default="default,warp,tex,hwtex")
ap.add_argument("--bp", default="tma,quad,tex,hwtex")
ap.add_argument("--out", default="")
a = ap.parse_args()

full = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
geom = full if a.views == 720 else tk.GeometryCone3D(full.volume_shape, full.volume_spacing, full.detector_shape,
                                                    full.detector_spacing, full.matrices[:: 720 // a.views][: a.views],
                                                    1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
step = 0.25
nvox = 512**3
V = geom.n_projections


def timed(fn):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(a.reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def rel(x, y):
    return float(torch.linalg.vector_norm((x - y).double()) / torch.linalg.vector_norm(y.double()))


res = {"views": V, "fp": {}, "bp": {}}
sino = torch.empty(geom.sinogram_shape, device="cuda")
ref_sino = None
for algo in a.fp.split(","):
    os.environ["TK_FP_ALGO"] = algo
    ms = timed(lambda: fp_tensor(vol, geom, step, out=sino))
    if ref_sino is None:
        ref_sino = sino.clone()
    res["fp"][algo] = {"ms": round(ms, 3), "gups": round(nvox * V / ms / 1e6, 2), "rel_vs_first": rel(sino, ref_sino)}
    print("fp", algo, res["fp"][algo], flush=True)
os.environ.pop("TK_FP_ALGO", None)

filt = filter_stage_tensor(ref_sino, geom, "shepp_logan")
out = torch.empty(geom.volume_shape, device="cuda")
ref_vol = None
for algo in a.bp.split(","):
    os.environ["TK_BP_ALGO"] = algo
    ms = timed(lambda: bp_tensor(filt, geom, True, out=out))
    if ref_vol is None:
        ref_vol = out.clone()
    res["bp"][algo] = {"ms": round(ms, 3), "gups": round(nvox * V / ms / 1e6, 2), "rel_vs_first": rel(out, ref_vol)}
    print("bp", algo, res["bp"][algo], flush=True)
print(json.dumps(res))
if a.out:
    Path(a.out).write_text(json.dumps(res, indent=1))
