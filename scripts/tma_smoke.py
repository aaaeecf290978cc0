"""Tiny TMA back-projection check against the quad kernel (run under a short timeout)."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2511_08427_b200 as tk
geom = tk.circular_cone_geometry((32, 32, 32), (1.0,) * 3, (48, 48), (1.5, 1.5), 12, 2 * math.pi, 1200.0, 750.0)
y = torch.randn(12, 48, 48, device="cuda")
os.environ["TK_BP_ALGO"] = "quad"
a = tk.back_project(tk.Sinogram(y, (1.5, 1.5)), geom, True).data
os.environ["TK_BP_ALGO"] = "tma"
b = tk.back_project(tk.Sinogram(y, (1.5, 1.5)), geom, True).data
torch.cuda.synchronize()
print("tma vs quad rel", float((a - b).norm() / a.norm()))
