"""Golden fixtures for the sinogram degradation simulators, made by importing the
REFERENCE's artifacts module (tomokit.artifacts, /root/reference/pkg/src) in the
build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_artifacts.py

Only the deterministic simulators are pinned bit-for-bit / to fp tolerance
(ring artifact, gantry-motion-blur kernels and convolutions); the random ones
(jitter, Poisson, Gaussian) have a distributional contract (artifacts.py:5-7)
and are tested statistically.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("TK_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, str(REF))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import tomokit as tk  # noqa: E402
from tomokit import artifacts as ta  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    rng = np.random.default_rng(20240917)
    out = {}
    for length in (3, 5, 9):
        for theta in (0.0, 0.3, np.pi / 4, 2.0, -1.1):
            out[f"kernel_{length}_{theta:.4f}"] = ta._line_kernel(length, theta)
    g = tk.circular_cone_geometry((16, 16, 16), (1, 1, 1), (20, 24), (1.0, 1.0), 8, 2 * np.pi, 1200.0, 750.0)
    s3 = rng.uniform(0.0, 3.0, (8, 20, 24))
    out["sino3"] = s3
    out["blur3_len5"] = ta.add_gantry_motion_blur(tk.Sinogram(s3, (1.0, 1.0)), g, 5).data
    out["blur3_len9"] = ta.add_gantry_motion_blur(tk.Sinogram(s3, (1.0, 1.0)), g, 9).data
    g2 = tk.GeometryParallel2D((16, 16), (1, 1), 40, 1.0, tk.circular_trajectory_2d(16, 2 * np.pi))
    s2 = rng.uniform(0.0, 3.0, (16, 40))
    out["sino2"] = s2
    out["blur2_len3"] = ta.add_gantry_motion_blur(tk.Sinogram(s2, (1.0,)), g2, 3).data
    out["ring3_zero"] = ta.add_ring_artifact(tk.Sinogram(s3, (1.0, 1.0)), [4, 17], (2, 6), "zero").data
    out["ring3_scale"] = ta.add_ring_artifact(tk.Sinogram(s3, (1.0, 1.0)), [0, 23], None, "scale", 0.7).data
    np.savez_compressed(OUT / "artifacts.npz", **out)
    print("wrote artifacts.npz:", ", ".join(sorted(out)))


if __name__ == "__main__":
    main()
