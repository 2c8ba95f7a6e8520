"""Times the two halves of the config-2 SVRG snapshot separately: the forward
over all 1800 angles (band kernel + reduction) and the plain gather over all
1800 angles, after a warm-up (CUDA events on the current stream)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, Projector, problems

size, A, B = 2048, 1800, 2900
proj = Projector(ParallelGeometry.uniform(A, B), size, size)
plan = proj.plan
x = torch.tensor(problems.ellipse_phantom(size, 60, 0), device="cuda", dtype=torch.float32)
y = torch.empty((A, B), device="cuda")
g = torch.empty_like(x)
for _ in range(5):
    plan.forward_into(x, y)
    plan.adjoint_into(y, g)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
n = 5
e[0].record()
for _ in range(n):
    plan.forward_into(x, y)
e[1].record()
for _ in range(n):
    plan.adjoint_into(y, g)
e[2].record()
torch.cuda.synchronize()
print(f"full forward {e[0].elapsed_time(e[1]) / n:.3f} ms, full gather {e[1].elapsed_time(e[2]) / n:.3f} ms")
