"""Kernel timings at the BASELINE sizes (CUDA events after a warm-up):
subset / full forward and gather at config 2, subset forward at configs 0/1,
FGP-100 at 2048^2 and the 3D FGP-100 at 256^3.

    python tools/kbench.py [fwd] [gather] [fgp] [fgp3]   (default: all)
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import ParallelGeometry, Projector, TvProxConfig, problems, tv_prox  # noqa
from paper_2602_09527_b200 import _native as N  # noqa: E402

want = set(sys.argv[1:]) or {"fwd", "gather", "fgp", "fgp3", "fwd3"}


def timed(fn, n, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(n):
        fn()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / n * 1e3  # us


def spin(sec=1.5):
    a = torch.randn(4096, 4096, device="cuda")
    torch.cuda.synchronize()
    t = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    t.record()
    while True:
        for _ in range(20):
            a = a @ a
            a = a / a.norm()
        e.record()
        torch.cuda.synchronize()
        if t.elapsed_time(e) > sec * 1e3:
            break


spin()
for name, (size, A, B, NS) in {"c2": (2048, 1800, 2900, 60), "c1": (512, 720, 768, 20),
                               "c0": (128, 180, 192, 10)}.items():
    g = ParallelGeometry.uniform(A, B)
    proj = Projector(g, size, size)
    plan = proj.plan
    x = torch.tensor(problems.ellipse_phantom(size, 60, 0), device="cuda", dtype=torch.float32)
    sub = tuple(range(0, A, NS))
    ys = torch.empty((len(sub), B), device="cuda")
    if "fwd" in want:
        f = timed(lambda: plan.forward_into(x, ys, sub), 50)
        line = f"{name} subset fwd {f:.1f} us"
        if name == "c2":
            y = torch.empty((A, B), device="cuda")
            line += f"  full fwd {timed(lambda: plan.forward_into(x, y, None), 5):.1f} us"
        print(line, flush=True)
    if "gather" in want and name != "c0":
        img = torch.empty_like(x)
        h = torch.zeros_like(x)
        fg = torch.zeros_like(x)
        xo = torch.empty_like(x)
        bad = torch.full((1,), 2**62, device="cuda", dtype=torch.int64)
        ep = N.StepEpilogue(3, 0, float(NS), 1e-7, 0.0, 0, N.ptr(x), N.ptr(h), N.ptr(fg), None,
                            N.ptr(xo), None, None, N.ptr(bad))
        hs = plan.selection(sub)

        def step():
            N.check(N.lib().pt_adjoint_step(plan.handle, hs, N.ptr(ys), ctypes.byref(ep),
                                            N.stream_handle()))
        line = f"{name} gather+step {timed(step, 50):.1f} us"
        if name == "c2":
            y = torch.randn((A, B), device="cuda")
            line += f"  full adj {timed(lambda: plan.adjoint_into(y, img, None), 5):.1f} us"
        print(line, flush=True)
    if "fgp" in want:
        cfg = TvProxConfig(alpha=0.02, inner_iterations=50 if name == "c0" else 100)
        out, st = tv_prox(x, 1.0, cfg)
        print(f"{name} fgp{cfg.inner_iterations} {timed(lambda: tv_prox(x, 1.0, cfg, warm=st), 10) / 1e3:.3f} ms",
              flush=True)
if "fwd3" in want:
    Z = 256
    vol = torch.tensor(problems.ellipsoid_phantom(Z, 40, 0), device="cuda", dtype=torch.float32)
    p3 = Projector(ParallelGeometry.uniform(360, 384), Z, Z, n_slices=Z)
    sub = tuple(range(0, 360, 40))
    y3 = torch.empty((len(sub), Z, 384), device="cuda")
    print(f"c3 subset fwd {timed(lambda: p3.plan.forward_into(vol, y3, sub), 30):.1f} us", flush=True)
if "fgp3" in want:
    Z = 256
    vol = torch.tensor(problems.ellipsoid_phantom(Z, 40, 0), device="cuda")
    p3 = Projector(ParallelGeometry.uniform(8, 8), Z, Z, n_slices=Z)
    cfg = TvProxConfig(alpha=0.05, inner_iterations=100)
    out, st = tv_prox(vol, 1.0, cfg)
    print(f"c3 fgp3d100 {timed(lambda: tv_prox(vol, 1.0, cfg, warm=st), 5) / 1e3:.3f} ms",
          flush=True)
