"""Full-angle forward and adjoint at c2 size (the SVRG snapshot's two
operators), per-angle cost against the subset operators."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, Projector, problems  # noqa: E402

size, A, B, NS = 2048, 1800, 2900, 60
g = ParallelGeometry.uniform(A, B)
proj = Projector(g, size, size)
plan = proj.plan
x = torch.tensor(problems.ellipse_phantom(size, 60, 0), device="cuda", dtype=torch.float32)
y = torch.empty((A, B), device="cuda")
img = torch.empty_like(x)
sub = tuple(range(0, A, NS))
ys = torch.empty((len(sub), B), device="cuda")


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(n):
        fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / n


for _ in range(20):
    plan.forward_into(x, ys, sub)
f_all = timed(lambda: plan.forward_into(x, y, None), 5)
a_all = timed(lambda: plan.adjoint_into(y, img, None), 5)
f_sub = timed(lambda: plan.forward_into(x, ys, sub), 20)
a_sub = timed(lambda: plan.adjoint_into(ys, img, sub), 20)
print(f"full fwd {f_all:.3f} ms ({f_all / A * 1e3:.2f} us/angle)  full adj {a_all:.3f} ms "
      f"({a_all / A * 1e3:.2f} us/angle)")
print(f"subset fwd {f_sub * 1e3:.1f} us ({f_sub / len(sub) * 1e3:.2f} us/angle)  subset adj "
      f"{a_sub * 1e3:.1f} us ({a_sub / len(sub) * 1e3:.2f} us/angle)")
