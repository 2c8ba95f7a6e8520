"""Small driver for ncu: one c2-size subset forward (SVRG difference), one
fused gather step and one FGP-100 prox call, via the C ABI."""
import ctypes
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, Projector, TvProxConfig, tv_prox, problems
from paper_2602_09527_b200 import _native as N

size, A, B, NS = 2048, 1800, 2900, 60
if len(sys.argv) > 1 and sys.argv[1] == "c1":
    size, A, B, NS = 512, 720, 768, 20
g = ParallelGeometry.uniform(A, B)
proj = Projector(g, size, size)
plan = proj.plan
x = torch.tensor(problems.ellipse_phantom(size, 60, 0), device="cuda", dtype=torch.float32)
x2 = 0.9 * x
sub = tuple(range(0, A, NS))
y = torch.empty((len(sub), B), device="cuda")
for _ in range(2):
    plan.forward_into(x, y, sub)
h = torch.zeros_like(x)
fg = torch.zeros_like(x)
xo = torch.empty_like(x)
bad = torch.full((1,), 2**62, device="cuda", dtype=torch.int64)
ep = N.StepEpilogue(3, 0, float(NS), 1e-7, 0.0, 0, N.ptr(x), N.ptr(h), N.ptr(fg), None,
                    N.ptr(xo), None, None, N.ptr(bad))
for _ in range(2):
    N.check(N.lib().pt_adjoint_step(plan.handle, plan.selection(sub), N.ptr(y), ctypes.byref(ep),
                                    N.stream_handle()))
cfg = TvProxConfig(alpha=0.02, inner_iterations=100)
out, st = tv_prox(x, 1.0, cfg)
# warm the GPU clocks before timing (short runs otherwise see the ramp)
for _ in range(30):
    plan.forward_into(x, y, sub)
    N.check(N.lib().pt_adjoint_step(plan.handle, plan.selection(sub), N.ptr(y), ctypes.byref(ep),
                                    N.stream_handle()))
for _ in range(5):
    out, st = tv_prox(x, 1.0, cfg, warm=st)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(10):
    plan.forward_into(x, y, sub)
t1.record(); torch.cuda.synchronize(); print("fwd us", t0.elapsed_time(t1) * 100)
t0.record()
for _ in range(10):
    N.check(N.lib().pt_adjoint_step(plan.handle, plan.selection(sub), N.ptr(y), ctypes.byref(ep),
                                    N.stream_handle()))
t1.record(); torch.cuda.synchronize(); print("gather us", t0.elapsed_time(t1) * 100)
t0.record()
for _ in range(3):
    out, st = tv_prox(x, 1.0, cfg, warm=st)
t1.record(); torch.cuda.synchronize(); print("fgp100 ms", t0.elapsed_time(t1) / 3)
if "--check" in sys.argv:
    import oracle as O
    O.set_mode("fast")
    ref = O.forward_project(x.double().cpu().numpy(), g, sub)
    plan.forward_into(x, y, sub)
    got = y.double().cpu().numpy()
    print("fwd rel err", float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
print("ok")
