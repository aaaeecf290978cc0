"""cfg5 matched transposes for ncu: A^T y (fp32 vector reductions) on the helical 512^3 / 720 / 1024^2 scan.

    ncu ... python scripts/prof_adjoint.py [--det]"""
import argparse
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import fp_adjoint_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--det", action="store_true", help="deterministic fixed-point mode")
a = ap.parse_args()
mats = tk.helical_trajectory_3d(720, 4 * math.pi, 1200.0, 750.0, (1024, 1024), (0.6, 0.6), -64.0, 64.0)
geom = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), mats, 1200.0, 750.0)
y = torch.rand(geom.sinogram_shape, device="cuda")
fp_adjoint_tensor(y, geom, 0.25, deterministic=a.det)
torch.cuda.synchronize()
print("done")
