"""Device timing of the cfg4 forward projection launched whole, by view chunks and by
row-band chunks (ForwardProjectionPlan), without and with the overlapped D2H copies."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import ops  # noqa: E402
from paper_2511_08427_b200.projectors import FP_BAND_ROWS, ForwardProjectionPlan, fp_tensor  # noqa: E402

geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
sino = torch.empty(geom.sinogram_shape, device="cuda")
host = torch.empty(geom.sinogram_shape, pin_memory=True)
copy = torch.cuda.Stream()
comp = torch.cuda.current_stream()


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        copy.synchronize()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return round(best, 2)


def run(kind, chunks, d2h):
    def fn():
        with ForwardProjectionPlan(vol, geom) as plan:
            for a, b in chunks:
                if kind == "views":
                    plan.project(slice(a, b), sino[a:b], 0.25)
                else:
                    plan.project_rows(a, b, sino, 0.25)
                if d2h:
                    ev = torch.cuda.Event()
                    ev.record(comp)
                    copy.wait_event(ev)
                    if kind == "views":
                        with torch.cuda.stream(copy):
                            host[a:b].copy_(sino[a:b], non_blocking=True)
                    else:
                        ops._copy_rows(host, sino, a, b, copy)
    return fn


res = {"whole": timed(lambda: fp_tensor(vol, geom, 0.25, out=sino))}
vch = ops._tapered(720, 12, 8, head=False, align=8)
rch = [(a * 8, b * 8) for a, b in ops._chunks(128, 12)]
res["views_12"] = timed(run("views", vch, False))
res["rows_12"] = timed(run("rows", rch, False))
res["views_12_d2h"] = timed(run("views", vch, True))
res["rows_12_d2h"] = timed(run("rows", rch, True))
res["rows_1"] = timed(run("rows", [(0, 1024)], False))
(_, first, runs) = ops._fp_row_schedule(geom, 0.25, 12)
sch = [(a * FP_BAND_ROWS, min(1024, b * FP_BAND_ROWS)) for a, b in [first] + runs]
res["schedule"] = sch
res["sched"] = timed(run("rows", sch, False))
res["sched_d2h"] = timed(run("rows", sch, True))
hostvol = torch.empty(geom.volume_shape, pin_memory=True)
scratch = torch.empty(geom.volume_shape, device="cuda")
(a0, b0), _, _ = ops._fp_row_schedule(geom, 0.25, 12)


def split(h2d):
    def fn():
        with ForwardProjectionPlan(vol, geom) as plan:
            if h2d:
                copy.wait_stream(comp)
                with torch.cuda.stream(copy):
                    scratch[:a0].copy_(hostvol[:a0], non_blocking=True)
                    scratch[b0:].copy_(hostvol[b0:], non_blocking=True)
            plan.cells(a0, b0)
            for i, (a, b) in enumerate(sch):
                if i == 1:
                    plan.cells(0, 512)
                plan.project_rows(a, b, sino, 0.25)
    return fn


res["sched_split"] = timed(split(False))
res["sched_split_h2d"] = timed(split(True))
firsts = {}
for name, f in (("first_alone", lambda: None),):
    pass


def first_only(h2d):
    def fn():
        with ForwardProjectionPlan(vol, geom) as plan:
            if h2d:
                copy.wait_stream(comp)
                with torch.cuda.stream(copy):
                    scratch[:a0].copy_(hostvol[:a0], non_blocking=True)
                    scratch[b0:].copy_(hostvol[b0:], non_blocking=True)
            plan.cells(0, 512)
            plan.project_rows(*sch[0], sino, 0.25)
    return fn


res["first_run"] = timed(first_only(False))
res["first_run_h2d"] = timed(first_only(True))
print(json.dumps(res))
