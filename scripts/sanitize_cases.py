#!/usr/bin/env python3
"""Small cfg3-shaped cases of every libtkb200 kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python scripts/sanitize_cases.py fp bp fpt bpt filter 2d
    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py bp filter
    compute-sanitizer --tool synccheck python scripts/sanitize_cases.py bp

Cases (shapes keep the sanitizer run to seconds; geometry = cfg3's circular
orbit scaled down: sdd 1200 / sid 750, detector wider than the volume's shadow
so clipped, missed and edge rays all occur):
  fp      forward projection: z-mirror-pair kernel (circular), the general
          z-fastest kernel (TK_FP_MIRROR=0), a helical orbit, an odd detector
  bp      back projection: TMA kernel (weighted / unweighted, odd volume),
          quad kernel (detector width not a multiple of 4), a row band / z-slab
  fpt     matched forward transpose, fp32 atomics and 64-bit fixed point
  bpt     matched back-projection transpose
  filter  FFT row filter (cone FDK filter stage), full detector and a row band
  2d      parallel / fan FP, BP, weighted BP, FBP and the 2D transposes
Each case prints a checksum; the parity of these paths is the GPU test suite's job.
"""

from __future__ import annotations

import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2511_08427_b200 as tk  # noqa: E402
from paper_2511_08427_b200 import projectors as P  # noqa: E402
from paper_2511_08427_b200 import filters as F  # noqa: E402


def vol3(n, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.rand(n, generator=g).cuda()


def circ(n=(48, 48, 48), det=(72, 76), views=24):
    return tk.circular_cone_geometry(n, (1.0, 1.0, 1.0), det, (1.6, 1.6), views, 2 * math.pi, 1200.0, 750.0)


def report(name, t):
    torch.cuda.synchronize()
    print(f"{name}: sum {float(t.double().sum()):.6e}", flush=True)


def case_fp():
    g = circ()
    x = vol3(g.volume_shape)
    print("path", P.forward_kernel_path(g))
    report("fp mirror", P.fp_tensor(x, g, 0.5))
    os.environ["TK_FP_MIRROR"] = "0"
    report("fp z-fastest", P.fp_tensor(x, g, 0.5))
    del os.environ["TK_FP_MIRROR"]
    h = tk.GeometryCone3D((40, 44, 36), (1.0, 1.1, 0.9), (33, 50), (1.5, 1.7),
                          tk.helical_trajectory_3d(20, 2 * math.pi, 1200.0, 750.0, (33, 50), (1.5, 1.7), -10, 10),
                          1200.0, 750.0)
    report("fp helical", P.fp_tensor(vol3(h.volume_shape, 1), h, 0.45))
    g3 = circ((31, 33, 35), (41, 43), 7)
    report("fp odd", P.fp_tensor(vol3(g3.volume_shape, 2), g3, 0.5))


def case_bp():
    g = circ()
    y = vol3(g.sinogram_shape, 3)
    for w in (False, True):
        report(f"bp tma w={w}", P.bp_tensor(y, g, w))
    g3 = circ((31, 33, 35), (40, 44), 9)
    report("bp tma odd", P.bp_tensor(vol3(g3.sinogram_shape, 4), g3, True))
    g5 = circ((30, 30, 30), (41, 43), 9)  # width not a multiple of 4 -> quad kernel
    report("bp quad", P.bp_tensor(vol3(g5.sinogram_shape, 5), g5, True))
    os.environ["TK_BP_ALGO"] = "quad"
    report("bp quad forced", P.bp_tensor(y, g, True))
    del os.environ["TK_BP_ALGO"]
    rows = g.detector_shape[0]
    band = y[:, 10:rows - 10].contiguous()
    report("bp band", P.bp_cone_tensor_ex(band, g, True, 10, 8, 24))


def case_fpt():
    g = circ()
    y = vol3(g.sinogram_shape, 6)
    report("fpT fp32", P.fp_adjoint_tensor(y, g, 0.5, deterministic=False))
    report("fpT fixed", P.fp_adjoint_tensor(y, g, 0.5, deterministic=True))


def case_bpt():
    g = circ()
    report("bpT", P.bp_adjoint_tensor(vol3(g.volume_shape, 7), g, True))


def case_filter():
    g = circ((48, 48, 48), (72, 300), 12)
    y = tk.Sinogram(vol3(g.sinogram_shape, 8), g.detector_spacing)
    for k in ("ramp", "shepp_logan", "cosine"):
        report(f"filter {k}", F.filter_stage(y, g, k).data)


def case_2d():
    ang = np.linspace(0, np.pi, 30, endpoint=False)
    gp = tk.GeometryParallel2D((37, 41), (1.0, 1.0), 59, 1.0, ang)
    x = vol3(gp.volume_shape, 9)
    report("par fp", P.fp_tensor(x, gp, 0.5))
    s = vol3(gp.sinogram_shape, 10)
    report("par bp", P.bp_tensor(s, gp))
    report("par fbp", tk.fbp_parallel_2d(tk.Sinogram(s, (1.0,)), gp, "ramp").data)
    report("par fpT", P.fp_adjoint_tensor(s, gp, 0.5))
    gf = tk.GeometryFan2D((37, 41), (1.0, 1.0), 64, 1.6, np.linspace(0, 2 * np.pi, 30, endpoint=False),
                          sdd=1200.0, sid=750.0)
    report("fan fp", P.fp_tensor(x, gf, 0.5))
    s = vol3(gf.sinogram_shape, 11)
    report("fan bp", P.bp_tensor(s, gf))
    report("fan bp w", P.bp_tensor(s, gf, True))
    report("fan fpT", P.fp_adjoint_tensor(s, gf, 0.5))


CASES = {"fp": case_fp, "bp": case_bp, "fpt": case_fpt, "bpt": case_bpt, "filter": case_filter, "2d": case_2d}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
