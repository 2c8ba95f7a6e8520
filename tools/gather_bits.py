"""Adjoint outputs for a bitwise A/B of two library builds (PT_LIB_OVERRIDE):
subset and full adjoints at the config-2/1/0 shapes (two-tap) and a
fine-detector geometry (several candidate bins per pixel)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, back_project  # noqa: E402

out = {}
rng = np.random.default_rng(0)
for name, (A, B, n, sub_step) in {"c2": (1800, 2900, 2048, 60), "c1": (720, 768, 512, 20),
                                  "c0": (180, 192, 128, 10), "fine": (90, 700, 160, 3)}.items():
    g = ParallelGeometry.uniform(A, B)
    y = torch.tensor(rng.standard_normal((A, B)), dtype=torch.float32, device="cuda")
    sub = tuple(range(1, A, sub_step))
    out[name + "_sub"] = back_project(y[list(sub)], g, (n, n), sub).cpu().numpy()
    out[name + "_full"] = back_project(y, g, (n, n)).cpu().numpy()
np.savez(sys.argv[1], **out)
