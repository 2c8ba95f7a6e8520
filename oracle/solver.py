"""Float64 CPU restatement of the ProxSkip-VR loop -- TEST INFRASTRUCTURE ONLY.

Restates, in numpy on top of the C oracle projector / FGP:
  * estimators  pkg/src/proxtomo/estimators.py:29-162
  * _init_state, _gradient_estimate, proxskip_step, _run_loop, run
                pkg/src/proxtomo/solvers.py:159-336
with the same PCG64 streams, draw order, pass accounting and row schedule.
Used (a) as the parity checker for configs the reference cannot run whole
(2048^2, 3D: its explicit CSR needs ~215 GB), after being pinned against
the reference's own runs (tests/golden/reference_*.npz), and (b) as the
timed CPU baseline of bench.py (kind "port", all host cores).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import OracleProjector, TvDual, tv_prox, tv_value


@dataclass
class Result:
    image: np.ndarray
    rows: list = field(default_factory=list)      # (passes, work_seconds, prox_calls, objective)
    iterations: list = field(default_factory=list)
    k: int = 0
    prox_calls: int = 0
    work_seconds: float = 0.0
    diverged_at: int | None = None
    cum_seconds: list = field(default_factory=list)  # work_seconds after each iteration


def partition(n_angles, n_subsets):
    """geometry.py:75-82."""
    return [tuple(range(k, n_angles, n_subsets)) for k in range(n_subsets)]


def objective(projector, data, x, alpha):
    """solvers.py:271-277."""
    r = projector.forward(x) - data
    val = 0.5 * float(np.sum(r * r))
    if alpha:
        val += alpha * tv_value(x)
    return val


def run_proxskip(projector: OracleProjector, data, *, gamma, p, estimator, n_subsets,
                 max_data_passes, seed=0, tv_alpha=None, tv_inner=10, warm_start=True,
                 nonneg=True, x0=None, record_objective=False, max_iterations=None,
                 max_seconds=None) -> Result:
    data = np.asarray(data, dtype=np.float64)
    shape = projector.shape
    x = np.zeros(shape) if x0 is None else np.array(x0, dtype=np.float64)
    h = np.zeros(shape)
    streams = np.random.SeedSequence(seed).spawn(3)
    rng_sub, rng_th, rng_rf = (np.random.default_rng(s) for s in streams)
    subsets = partition(projector.geometry.n_angles, n_subsets) if estimator != "full" else None
    n = n_subsets

    def sub_grad(z, i):
        s = subsets[i]
        return projector.adjoint(projector.forward(z, s) - data[list(s)], s)

    def full_grad(z):
        return projector.adjoint(projector.forward(z) - data)

    passes = 0.0
    table = total = snap = fg = None
    since = 0
    if estimator == "saga":
        table = np.zeros((n,) + tuple(shape))
        total = np.zeros(shape)
    elif estimator in ("svrg", "lsvrg"):
        snap = x.copy()
        fg = full_grad(snap)
        passes += 1.0
    warm = None
    res = Result(image=x)

    def log(k):
        obj = objective(projector, data, x, tv_alpha) if record_objective else None
        res.rows.append((passes, res.work_seconds, res.prox_calls, obj))
        res.iterations.append(k)

    log(0)
    last_floor = math.floor(passes + 1e-12)
    k = 0
    while True:
        t0 = time.perf_counter()
        # ---- _gradient_estimate (solvers.py:189-214) ----
        if estimator == "full":
            g = full_grad(x)
            ch = 1.0
        elif estimator in ("sgd", "saga"):
            i = int(rng_sub.integers(n))
            gi = sub_grad(x, i)
            if estimator == "sgd":
                g = n * gi
            else:
                old = table[i]
                g = n * gi + (total - n * old)
                total = (total - old) + gi
                table[i] = gi
            ch = 1.0 / n
        else:
            c = 0.0
            if estimator == "svrg":
                refresh = since >= n
            else:
                refresh = True if 1.0 / n >= 1.0 else bool(rng_rf.random() < 1.0 / n)
            if refresh:
                snap = x.copy()
                fg = full_grad(snap)
                since = 0
                c += 1.0
            i = int(rng_sub.integers(n))
            g = n * (sub_grad(x, i) - sub_grad(snap, i)) + fg
            since += 1
            ch = c + 2.0 / n
        # ---- proxskip_step (solvers.py:230-254) ----
        base = x - gamma * g
        x_hat = base + gamma * h
        theta = True if p >= 1.0 else bool(rng_th.random() < p)
        if theta:
            target = base + (gamma - gamma / p) * h
            if tv_alpha:
                x_next, warm = tv_prox(target, gamma / p, tv_alpha, tv_inner, nonneg,
                                       warm if warm_start else None)
            else:
                x_next = target
            res.prox_calls += 1
        else:
            x_next = x_hat
        if not np.all(np.isfinite(x_next)):
            res.diverged_at = k
            res.image = None
            return res
        if theta:
            h = h + (p / gamma) * (x_next - x_hat)
        x = x_next
        k += 1
        passes += ch
        res.work_seconds += time.perf_counter() - t0
        res.cum_seconds.append(res.work_seconds)
        exhausted = passes >= max_data_passes - 1e-9
        if max_iterations is not None and k >= max_iterations:
            exhausted = True
        if max_seconds is not None and res.work_seconds >= max_seconds:
            exhausted = True
        crossed = math.floor(passes + 1e-12) > last_floor
        if crossed or exhausted:
            last_floor = math.floor(passes + 1e-12)
            log(k)
            if exhausted:
                break
    res.image = x
    res.k = k
    return res


def run_fista(projector, data, *, gamma, max_data_passes, tv_alpha=None, tv_inner=10,
              warm_start=True, nonneg=True, accelerate=True, record_objective=False) -> Result:
    """run_fista / run_ista (solvers.py:339-392): full gradient at y, prox every
    iteration, t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2, y = x+ + ((t_k - 1) / t_{k+1})
    (x+ - x); one data pass per iteration, rows as _run_loop (:280-324)."""
    data = np.asarray(data, dtype=np.float64)
    x = np.zeros(projector.shape)
    y = x.copy()
    t = 1.0
    warm = None
    passes = 0.0
    res = Result(image=x)

    def log(k):
        obj = objective(projector, data, x, tv_alpha) if record_objective else None
        res.rows.append((passes, res.work_seconds, res.prox_calls, obj))
        res.iterations.append(k)

    log(0)
    last_floor = math.floor(passes + 1e-12)
    k = 0
    while True:
        t0 = time.perf_counter()
        grad = projector.adjoint(projector.forward(y) - data)
        target = y - gamma * grad
        if tv_alpha:
            x_next, warm = tv_prox(target, gamma, tv_alpha, tv_inner, nonneg,
                                   warm if warm_start else None)
        else:
            x_next = target
        res.prox_calls += 1
        if not np.all(np.isfinite(x_next)):
            res.diverged_at = k
            res.image = None
            return res
        if accelerate:
            t_next = (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0
            y = x_next + ((t - 1.0) / t_next) * (x_next - x)
            t = t_next
        else:
            y = x_next
        x = x_next
        k += 1
        passes += 1.0
        res.work_seconds += time.perf_counter() - t0
        exhausted = passes >= max_data_passes - 1e-9
        crossed = math.floor(passes + 1e-12) > last_floor
        if crossed or exhausted:
            last_floor = math.floor(passes + 1e-12)
            log(k)
            if exhausted:
                break
    res.image = x
    res.k = k
    return res


def _forward_diff(x):
    """regularizers.py:62-68: forward differences, 0 on the last row / column."""
    gv = np.zeros_like(x)
    gh = np.zeros_like(x)
    gv[:-1, :] = x[1:, :] - x[:-1, :]
    gh[:, :-1] = x[:, 1:] - x[:, :-1]
    return gv, gh


def _diff_adjoint(a, b):
    """regularizers.py:71-76: D^T(a, b) using only the [:-1] parts."""
    out = np.zeros_like(a)
    out[:-1, :] -= a[:-1, :]
    out[1:, :] += a[:-1, :]
    out[:, :-1] -= b[:, :-1]
    out[:, 1:] += b[:, :-1]
    return out


def run_pdhg(projector, data, n_iterations, alpha=0.0, nonneg=False, snapshot_at=None):
    """Diagonally preconditioned PDHG (solvers.py:395-455), float64."""
    data = np.asarray(data, dtype=np.float64)
    shape = projector.shape
    row_sums = projector.forward(np.ones(shape))
    with np.errstate(divide="ignore"):
        sigma_a = np.where(row_sums > 0.0, 1.0 / row_sums, 0.0)
    col_sums = projector.adjoint(np.ones_like(data))
    if alpha > 0.0:
        dc = np.zeros(shape)
        dc[:-1, :] += 1.0
        dc[1:, :] += 1.0
        dc[:, :-1] += 1.0
        dc[:, 1:] += 1.0
        col_sums = col_sums + dc
    tau = 1.0 / np.maximum(col_sums, 1e-12)
    sigma_d = 0.5
    x = np.zeros(shape)
    x_bar = x.copy()
    y = np.zeros_like(data)
    zv = np.zeros(shape)
    zh = np.zeros(shape)
    snapshot = None
    for it in range(1, n_iterations + 1):
        y = (y + sigma_a * (projector.forward(x_bar) - data)) / (1.0 + sigma_a)
        ascent = projector.adjoint(y)
        if alpha > 0.0:
            gv, gh = _forward_diff(x_bar)
            zv = zv + sigma_d * gv
            zh = zh + sigma_d * gh
            scale = np.maximum(1.0, np.sqrt(zv * zv + zh * zh) / alpha)
            zv /= scale
            zh /= scale
            ascent = ascent + _diff_adjoint(zv, zh)
        x_old = x
        x = x - tau * ascent
        if nonneg:
            np.maximum(x, 0.0, out=x)
        x_bar = 2.0 * x - x_old
        if snapshot_at is not None and it == snapshot_at:
            snapshot = x.copy()
    return (x, snapshot) if snapshot_at is not None else x
