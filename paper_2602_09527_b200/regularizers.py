"""Isotropic TV: value and FGP proximal map on the GPU.

Drop-in for pkg/src/proxtomo/regularizers.py:32-133 (``TvProxConfig``,
``TvDualState``, ``tv_value``, ``nonneg_prox``, ``tv_prox``).  The FGP inner
loop runs in the temporally blocked sm_100a kernel (csrc/fgp.cu); a 3D
volume (Z, H, W) uses the slice-stacked 3D extension (third dual w, dual
step 1/(12 lam)).  Plug-and-play denoisers (:136-202) are out of scope
(DESIGN.md).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _native as N
from .geometry import ParallelGeometry
from .projector import as_device, get_plan

_GRID_GEOMETRY = ParallelGeometry((0.0,), 1)


def grid_plan(shape):
    """A plan that only carries the image grid (FGP / TV kernels)."""
    shape = tuple(int(s) for s in shape)
    z = shape[0] if len(shape) == 3 else 1
    return get_plan(_GRID_GEOMETRY, shape[-1], shape[-2], z)


@dataclass(frozen=True)
class TvProxConfig:
    """TV weight plus the inner FGP iteration budget (regularizers.py:32-45)."""

    alpha: float
    inner_iterations: int = 10
    warm_start: bool = True
    nonneg: bool = True

    def __post_init__(self):
        if self.alpha <= 0.0:
            raise ValueError("alpha must be positive")
        if self.inner_iterations < 1:
            raise ValueError("inner_iterations must be >= 1")


@dataclass
class TvDualState:
    """FGP duals carried across warm-started calls (regularizers.py:48-59);
    ``w`` is the third dual of the 3D prox."""

    p: torch.Tensor
    q: torch.Tensor
    weight: float
    w: torch.Tensor | None = None


def tv_value(image) -> float:
    """Isotropic TV, forward differences, replicate boundary (regularizers.py:79-82)."""
    x = as_device(image)
    plan = grid_plan(x.shape)
    out = torch.empty(N.PT_RED_DOUBLES, device="cuda", dtype=torch.float64)
    N.check(N.lib().pt_tv_value(plan.handle, N.ptr(x), N.ptr(out), N.stream_handle()), "tv_value")
    return float(out[0].item())


def nonneg_prox(image) -> torch.Tensor:
    """Projection onto the nonnegative orthant (regularizers.py:85-87)."""
    return torch.clamp_min(as_device(image), 0.0)


def tv_prox(image, tau: float, config: TvProxConfig,
            warm: TvDualState | None = None) -> tuple[torch.Tensor, TvDualState]:
    """Proximal map of tau*alpha*TV (+ nonnegativity) by exactly
    ``config.inner_iterations`` FGP iterations (regularizers.py:90-133).

    Warm duals are reused iff their shape matches and their weight equals
    tau*alpha to relative 1e-12 (:102-106); momentum restarts every call."""
    if tau <= 0.0:
        raise ValueError("tau must be positive")
    v = as_device(image)
    if v.ndim not in (2, 3):
        raise ValueError(f"image must be 2D or 3D, got shape {tuple(v.shape)}")
    lam = tau * config.alpha
    use_warm = (warm is not None and tuple(warm.p.shape) == tuple(v.shape)
                and abs(warm.weight - lam) <= 1e-12 * abs(lam))
    if use_warm:
        p, q = as_device(warm.p).clone(), as_device(warm.q).clone()
        w = as_device(warm.w).clone() if (v.ndim == 3 and warm.w is not None) else None
    else:
        p, q, w = torch.zeros_like(v), torch.zeros_like(v), None
    if v.ndim == 3 and w is None:
        w = torch.zeros_like(v)
    plan = grid_plan(v.shape)
    out = torch.empty_like(v)
    N.check(N.lib().pt_tv_prox(plan.handle, N.ptr(v), float(lam), int(config.inner_iterations),
                               int(bool(config.nonneg)), N.ptr(p), N.ptr(q), N.ptr(w), N.ptr(out),
                               None, None, 0.0, 0, None, N.ptr(plan.fgp_work()),
                               N.stream_handle()), "tv_prox")
    return out, TvDualState(p=p, q=q, weight=lam, w=w)
