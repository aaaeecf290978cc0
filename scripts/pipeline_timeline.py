"""Timelines of the pinned-host pipelines at cfg4 -- py_fbp (ops._fdk_cone_overlapped) and
py_forward_project (ops._fp_cone_overlapped): CUDA events on the copy and compute streams
around every chunk's copy, filter, back projection and projection, to locate the time the
boundary calls spend beyond the device-resident operators.

    python scripts/pipeline_timeline.py [fdk|fp ...]
"""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import filters as F  # noqa: E402
from paper_2511_08427_b200 import ops  # noqa: E402
from paper_2511_08427_b200 import projectors as P  # noqa: E402

cfg = {"geometry_kind": "cone3d", "volume_shape": [512] * 3, "volume_spacing": [0.5] * 3,
       "detector_shape": [1024, 1024], "detector_spacing": [0.6, 0.6], "number_of_projections": 720,
       "angular_range": 2 * math.pi, "sdd": 1200.0, "sid": 750.0, "filter_kind": "shepp_logan"}
geom = ops.PipelineConfig.from_dict(cfg).build_geometry()
host = torch.empty(geom.sinogram_shape, pin_memory=True)
host.uniform_()

marks = []
orig_filter, orig_bp = F.filter_stage_tensor, P.bp_cone_tensor_ex
orig_project = P.ForwardProjectionPlan.project
orig_copy = torch.Tensor.copy_


def ev(tag):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((tag, e))


def filt(*a, **k):
    ev("filter>")
    r = orig_filter(*a, **k)
    ev("filter<")
    return r


def bp(*a, **k):
    ev("bp>")
    r = orig_bp(*a, **k)
    ev("bp<")
    return r


def project(self, *a, **k):
    ev("fp>")
    r = orig_project(self, *a, **k)
    ev("fp<")
    return r


def copy_(self, src, non_blocking=False):
    ev(f"copy> {tuple(self.shape)[:1]} {'h2d' if self.is_cuda else 'd2h'}")
    r = orig_copy(self, src, non_blocking=non_blocking)
    ev("copy<")
    return r


vol = torch.empty(geom.volume_shape, pin_memory=True)
vol.uniform_()
for op in sys.argv[1:] or ["fdk", "fp"]:
    for rep in range(2):
        marks.clear()
        F.filter_stage_tensor, P.bp_cone_tensor_ex = filt, bp
        P.ForwardProjectionPlan.project = project
        torch.Tensor.copy_ = copy_
        torch.cuda.synchronize()
        ev("start")
        if op == "fdk":
            ops.py_fbp(host, cfg)
        else:
            ops.py_forward_project(vol, cfg)
        torch.cuda.synchronize()
        torch.Tensor.copy_ = orig_copy
        P.ForwardProjectionPlan.project = orig_project
        F.filter_stage_tensor, P.bp_cone_tensor_ex = orig_filter, orig_bp
    t0 = marks[0][1]
    rows = [(tag, round(t0.elapsed_time(e), 2)) for tag, e in marks]
    print("==", op)
    for r in rows:
        print(r)
    print(json.dumps({"op": op, "total_ms": max(t for _, t in rows)}))
