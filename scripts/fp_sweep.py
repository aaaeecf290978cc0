"""Sweep environment-selected kernel configurations of one operator at cfg4.

    python scripts/fp_sweep.py --op fp --configs "TK_FP_MIRROR=0;TK_FP_MIRROR=1,TK_FP_CFG=6x2"
    python scripts/fp_sweep.py --op bp --configs "TK_BP_ALGO=tma;TK_BP_ALGO=quad"
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
from paper_2511_08427_b200.filters import filter_stage_tensor  # noqa: E402
from paper_2511_08427_b200.projectors import bp_tensor, fp_tensor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="fp")
ap.add_argument("--configs", required=True)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--views", type=int, default=720)
a = ap.parse_args()

full = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
geom = full if a.views == 720 else tk.GeometryCone3D(full.volume_shape, full.volume_spacing, full.detector_shape,
                                                    full.detector_spacing, full.matrices[:: 720 // a.views][: a.views],
                                                    1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
sino = torch.empty(geom.sinogram_shape, device="cuda")
fp_tensor(vol, geom, 0.25, out=sino)
filt = filter_stage_tensor(sino, geom, "shepp_logan") if a.op in ("bp", "filter") else None
out = torch.empty(geom.volume_shape, device="cuda")
ref = None
res = {}
for cfg in a.configs.split(";"):
    env = dict(kv.split("=") for kv in cfg.split(",") if kv)
    os.environ.update(env)
    if a.op == "fp":
        fn = lambda: fp_tensor(vol, geom, 0.25, out=sino)  # noqa: E731
    elif a.op == "filter":
        fn = lambda: filter_stage_tensor(sino, geom, "shepp_logan", out=filt)  # noqa: E731
    else:
        fn = lambda: bp_tensor(filt, geom, True, out=out)  # noqa: E731
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
    res_t = {"fp": sino, "filter": filt}.get(a.op, out)
    if ref is None:
        ref = res_t.clone()
    err = float(torch.linalg.vector_norm((res_t - ref).double()) / torch.linalg.vector_norm(ref.double()))
    res[cfg] = {"ms": round(best, 3), "rel_vs_first": err}
    print(a.op, cfg, res[cfg], flush=True)
    for k in env:
        del os.environ[k]
print(json.dumps(res))
