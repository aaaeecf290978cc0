"""Does a concurrent D2H copy slow the forward projector?  FP time alone, with a
contiguous (1D) D2H of 3 GB on another stream, and with the same bytes as a pitched
(2D, tk_copy_2d) copy, and as per-view 1D row-band copies."""
import json
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import ops  # noqa: E402
from paper_2511_08427_b200.projectors import fp_tensor  # noqa: E402

geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
vol = tk.phantoms.shepp_logan_3d(geom.volume_shape)
sino = torch.empty(geom.sinogram_shape, device="cuda")
other = torch.rand(geom.sinogram_shape, device="cuda")
host = torch.empty(geom.sinogram_shape, pin_memory=True)
copy = torch.cuda.Stream()
comp = torch.cuda.current_stream()


def fp_with(copier):
    fp_tensor(vol, geom, 0.25, out=sino)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    copy.wait_stream(comp)
    s.record(comp)
    if copier:
        copier()
    fp_tensor(vol, geom, 0.25, out=sino)
    e.record(comp)
    torch.cuda.synchronize()
    return round(s.elapsed_time(e), 2)


def c1d():
    with torch.cuda.stream(copy):
        host.copy_(other, non_blocking=True)


def c2d():
    for r in range(0, 1024, 128):
        ops._copy_rows(host, other, r, r + 128, copy)


def cviews():
    with torch.cuda.stream(copy):
        for r in range(0, 1024, 128):
            for v in range(720):
                host[v, r:r + 128].copy_(other[v, r:r + 128], non_blocking=True)


res = {}
for name, fn in [("alone", None), ("d2h_1d", c1d), ("d2h_2d", c2d), ("d2h_per_view", cviews), ("alone2", None)]:
    res[name] = fp_with(fn)
print(json.dumps(res))
