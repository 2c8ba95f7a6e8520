"""Times the config-2 projector launches whose CTA grain is tunable (PT_FWD_WAVES /
PT_FWD_GROUPS for the band forward, PT_GATHER_TILE for the gather): one subset
forward, one subset gather, the full 1800-angle forward and the full gather.
CUDA events on the current stream after a warm-up; prints one line of us."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, Projector, problems

size, A, B, NS = 2048, 1800, 2900, 60
proj = Projector(ParallelGeometry.uniform(A, B), size, size)
plan = proj.plan
x = torch.tensor(problems.ellipse_phantom(size, 60, 0), device="cuda", dtype=torch.float32)
sub = tuple(range(0, A, NS))
ys = torch.empty((len(sub), B), device="cuda")
y = torch.empty((A, B), device="cuda")
g = torch.empty_like(x)


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000.0 / n


for _ in range(20):  # clocks up
    plan.forward_into(x, y)
res = {
    "fwd_sub": timed(lambda: plan.forward_into(x, ys, sub), 50),
    "adj_sub": timed(lambda: plan.adjoint_into(ys, g, sub), 50),
    "fwd_full": timed(lambda: plan.forward_into(x, y), 10),
    "adj_full": timed(lambda: plan.adjoint_into(y, g), 10),
}
env = {k: v for k, v in os.environ.items() if k.startswith("PT_")}
print(env, " ".join(f"{k}={v:.1f}" for k, v in res.items()), flush=True)
