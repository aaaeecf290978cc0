"""One cfg4 step (forward projection + FDK) for ncu: `ncu ... python scripts/prof_step.py`.

--views N limits the orbit to N views (same geometry, fewer launches' worth of work)."""

import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.filters import fdk_tensor  # noqa: E402
from paper_2511_08427_b200.projectors import fp_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--views", type=int, default=720)
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--det", type=int, default=1024)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--what", default="fp,fdk")
a = ap.parse_args()

full = tk.circular_cone_geometry((a.n,) * 3, (256 / a.n,) * 3, (a.det, a.det), (614.4 / a.det,) * 2, 720,
                                 2 * math.pi, 1200.0, 750.0)
geom = full if a.views == 720 else tk.GeometryCone3D(full.volume_shape, full.volume_spacing,
                                                    full.detector_shape, full.detector_spacing,
                                                    full.matrices[:: 720 // a.views][: a.views], 1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
step = 0.5 * min(geom.volume_spacing)
sino = torch.empty(geom.sinogram_shape, device="cuda")
work = torch.empty_like(sino)
out = torch.empty(geom.volume_shape, device="cuda")
fp_tensor(vol, geom, step, out=sino)
for _ in range(a.reps):
    if "fp" in a.what:
        fp_tensor(vol, geom, step, out=sino)
    if "fdk" in a.what:
        fdk_tensor(sino, geom, "shepp_logan", workspace=work, out=out)
torch.cuda.synchronize()
print("done", float(out.abs().mean()))
