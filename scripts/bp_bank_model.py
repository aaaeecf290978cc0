"""Shared-memory bank-conflict model of the TMA back projector's tap gathers (cfg4).

For sampled (view, 16x16x32 block) pairs it reproduces the kernel's per-lane detector
coordinates, the TMA box origin and the tile address of each of the four taps, and
counts LDS wavefronts per warp instruction (max distinct addresses in one bank) for a
given tile pitch bw and warp shape (WX x WY voxel columns).  CPU only (numpy).

    python scripts/bp_bank_model.py
"""

import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2511_08427_b200 as tk  # noqa: E402

geom = tk.circular_cone_geometry((512,) * 3, (0.5,) * 3, (1024, 1024), (0.6, 0.6), 720, 2 * math.pi, 1200.0, 750.0)
mats = geom.matrix_array()
n, R, C = 512, 1024, 1024
cu, cv = (C - 1) / 2.0, (R - 1) / 2.0
s = 0.5
c0v = (n - 1) / 2.0


def lanes_rc(P, bx, by, bz, wx0, wy0, WX, WY, k):
    tx = np.arange(32) % WX
    ty = np.arange(32) // WX
    ix = bx * 16 + wx0 + tx
    iy = by * 16 + wy0 + ty
    iz = bz * 32 + k
    X = (ix - c0v) * s
    Y = (iy - c0v) * s
    Z = (iz - c0v) * s
    h = P @ np.stack([X, Y, np.full(32, Z), np.ones(32)])
    return h[1] / h[2], h[0] / h[2]  # row, col


def box_origin(P, bx, by, bz):
    xs = [(bx * 16 - c0v) * s, (bx * 16 + 15 - c0v) * s]
    ys = [(by * 16 - c0v) * s, (by * 16 + 15 - c0v) * s]
    zs = [(bz * 32 - c0v) * s, (bz * 32 + 31 - c0v) * s]
    pts = np.array([[x, y, z, 1.0] for x in xs for y in ys for z in zs]).T
    h = P @ pts
    return int(math.floor((h[1] / h[2]).min())) - 1, (int(math.floor((h[0] / h[2]).min())) - 1) & ~3


def wavefronts(addr):
    banks = addr % 32
    w = 0
    for b in np.unique(banks):
        w = max(w, len(np.unique(addr[banks == b])))
    return w


def model(bw, WX, WY, views=range(0, 720, 45), blocks=((3, 5, 2), (16, 16, 8), (28, 9, 13), (10, 27, 5))):
    tot = cnt = 0
    for v in views:
        P = mats[v]
        for bx, by, bz in blocks:
            r0, cb0 = box_origin(P, bx, by, bz)
            for wy0 in range(0, 16, WY):
                for wx0 in range(0, 16, WX):
                    for k in range(0, 32, 4):
                        fr, fc = lanes_rc(P, bx, by, bz, wx0, wy0, WX, WY, k)
                        r = np.floor(fr).astype(int) - r0
                        c = np.floor(fc).astype(int) - cb0
                        for dr, dc in ((0, 0), (0, 1), (1, 0), (1, 1)):
                            tot += wavefronts((r + dr) * bw + c + dc)
                            cnt += 1
    return tot / cnt


if __name__ == "__main__":
    for WX, WY in ((16, 2), (8, 4), (32, 1), (4, 8)):
        for bw in (44, 48, 52, 56, 60, 64, 68, 72, 76, 80):
            print(f"warp {WX}x{WY} bw {bw}: {model(bw, WX, WY):.3f} wavefronts per LDS", flush=True)
