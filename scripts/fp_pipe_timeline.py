"""CUDA-event timeline of py_forward_project's upload-ordered row-band pipeline at cfg4
(events on the stream each step is issued to), wall time of the call, and the band runs."""
import json
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import ops  # noqa: E402
from paper_2511_08427_b200 import projectors as P  # noqa: E402

cfg = {"geometry_kind": "cone3d", "volume_shape": [512] * 3, "volume_spacing": [0.5] * 3,
       "detector_shape": [1024, 1024], "detector_spacing": [0.6, 0.6], "number_of_projections": 720,
       "angular_range": 2 * math.pi, "sdd": 1200.0, "sid": 750.0, "filter_kind": "shepp_logan"}
geom = ops.PipelineConfig.from_dict(cfg).build_geometry()
host = torch.empty(geom.volume_shape, pin_memory=True)
host.copy_(tk.phantoms.shepp_logan_3d(geom.volume_shape))
marks = []


def ev(tag, stream=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    marks.append((tag, e))


def wrap(obj, name, tag, stream_arg=None):
    orig = getattr(obj, name)

    def f(*a, **k):
        s = a[stream_arg] if stream_arg is not None else None
        ev(tag + ">", s)
        r = orig(*a, **k)
        ev(tag + "<", s)
        return r
    setattr(obj, name, f)


wrap(P.ForwardProjectionPlan, "project_rows", "fp")
wrap(P.ForwardProjectionPlan, "project", "fpv")
wrap(P.ForwardProjectionPlan, "cells", "cells")
wrap(ops, "_copy_rows", "d2h", stream_arg=4)
step = ops.PipelineConfig.from_dict(cfg).sampling().step(geom.volume_spacing)
print("bands:", P.band_z_extent(geom, step)[::8].tolist(), file=sys.stderr)
for it in range(3):
    marks.clear()
    torch.cuda.synchronize()
    ev("start")
    t0 = time.perf_counter()
    ops.py_forward_project(host, cfg)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
t0 = marks[0][1]
print(json.dumps({"wall_ms": round(wall, 2),
                  "events": [(tag, round(t0.elapsed_time(e), 2)) for tag, e in marks[1:]]}))
