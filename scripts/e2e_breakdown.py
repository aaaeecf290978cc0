"""Where the e2e step's time goes: py_forward_project (pinned host volume -> pinned host
sinogram) and py_fbp (pinned host sinogram -> pinned host volume) against the same
operators on device-resident data, cfg4, wall clock (host-synchronised) per phase."""
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import ops  # noqa: E402
from paper_2511_08427_b200.filters import fdk_tensor  # noqa: E402
from paper_2511_08427_b200.projectors import fp_tensor  # noqa: E402

cfg = {"geometry_kind": "cone3d", "volume_shape": [512] * 3, "volume_spacing": [0.5] * 3,
       "detector_shape": [1024, 1024], "detector_spacing": [0.6, 0.6], "number_of_projections": 720,
       "angular_range": 2 * math.pi, "sdd": 1200.0, "sid": 750.0, "filter_kind": "shepp_logan"}
geom = ops.PipelineConfig.from_dict(cfg).build_geometry()
vol = tk.phantoms.shepp_logan_3d((512,) * 3)
host_vol = torch.empty((512,) * 3, pin_memory=True)
host_vol.copy_(vol)


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return round(best * 1e3, 1), r


res = {}
res["h2d_volume_ms"], _ = wall(lambda: host_vol.to("cuda", non_blocking=True))
res["fp_device_ms"], sino = wall(lambda: fp_tensor(vol, geom, 0.25))
res["py_forward_project_ms"], host_sino = wall(lambda: ops.py_forward_project(host_vol, cfg))
res["fdk_device_ms"], _ = wall(lambda: fdk_tensor(sino, geom, "shepp_logan"))
res["h2d_sinogram_ms"], _ = wall(lambda: host_sino.to("cuda", non_blocking=True))
res["py_fbp_ms"], _ = wall(lambda: ops.py_fbp(host_sino, cfg))
res["e2e_step_ms"], _ = wall(lambda: ops.py_fbp(ops.py_forward_project(host_vol, cfg), cfg))
print(json.dumps(res))
