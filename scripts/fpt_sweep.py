"""cfg5 (helical 512^3 / 720 / 1024^2) matched forward transpose A^T y under env-selected variants.

    python scripts/fpt_sweep.py --configs "TK_FPT_CARRY=1;TK_FPT_CARRY=0" """
import argparse
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200.projectors import fp_adjoint_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", required=True)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
mats = tk.helical_trajectory_3d(720, 4 * math.pi, 1200.0, 750.0, (1024, 1024), (0.6, 0.6), -64.0, 64.0)
geom = tk.GeometryCone3D((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), mats, 1200.0, 750.0)
y = torch.rand(geom.sinogram_shape, device="cuda")
res, ref = {}, None
for cfg in a.configs.split(";"):
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    os.environ.update(env)
    det = env.get("DET") == "1"
    out = fp_adjoint_tensor(y, geom, 0.25, deterministic=det)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(a.reps):
        s.record()
        out = fp_adjoint_tensor(y, geom, 0.25, deterministic=det)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    if ref is None:
        ref = out.clone()
    err = float(torch.linalg.vector_norm((out - ref).double()) / torch.linalg.vector_norm(ref.double()))
    res[cfg] = {"ms": round(best, 2), "rel_vs_first": err}
    print(cfg, res[cfg], flush=True)
    for k in env:
        os.environ.pop(k, None)
print(json.dumps(res))
