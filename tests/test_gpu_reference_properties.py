"""The reference's own property tests, restated for the device implementation.

Each test mirrors one of proxtomo's unit tests (pkg/tests/test_projector.py,
test_estimators.py, test_regularizers.py, test_solvers.py; cited per test) on
the native path: the same invariant, with float32 tolerances where the
reference compares float64 bits of a different evaluation order, and bitwise
where the device evaluates the same float32 expression on both sides.
"""
import math

import numpy as np
import pytest
import torch

from paper_2602_09527_b200 import (ParallelGeometry, Projector, SolverConfig, TomoProblem,
                                   TvProxConfig, build_staggered_partition, composite_objective,
                                   problems, run, run_ista, run_pdhg_reference, tv_prox)
from paper_2602_09527_b200 import estimators as E
from paper_2602_09527_b200.solvers import RUN_COLUMNS, _init_state, proxskip_step

pytestmark = pytest.mark.gpu


def cpu(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def rel(a, b):
    return float(np.linalg.norm(cpu(a) - cpu(b)) / max(np.linalg.norm(cpu(b)), 1e-30))


@pytest.fixture(scope="module")
def small():
    g = ParallelGeometry.uniform(12, 23)
    proj = Projector(g, 16, 16)
    x_true = problems.ellipse_phantom(16, 3, 5)
    data = cpu(proj.forward(x_true)) + 0.01 * np.random.default_rng(5).standard_normal((12, 23))
    problem = TomoProblem(proj, data, tv=TvProxConfig(alpha=0.05, inner_iterations=10))
    return problem, proj, data, proj.norm_sq(80, 0)


# ---- projector (test_projector.py) ------------------------------------------

def test_subset_adjoints_sum_to_the_normal_operator(small):
    """sum_i A_i^T A_i x = A^T A x (test_projector.py: subset adjoints)."""
    _, proj, _, _ = small
    x = np.random.default_rng(1).random((16, 16))
    full = cpu(proj.adjoint(proj.forward(x)))
    part = build_staggered_partition(12, 4)
    acc = sum(cpu(proj.adjoint(proj.forward(x, s), s)) for s in part.subsets)
    assert rel(acc, full) <= 1e-6


def test_norm_sq_deterministic_monotone_and_below_the_dense_bound():
    """Power-iteration estimates: reproducible for a seed, non-decreasing in the
    iteration count, never above sigma_max^2 of the assembled matrix
    (test_projector.py: norm_sq_deterministic / monotone_lower_bound /
    matches_dense_svd)."""
    g = ParallelGeometry.uniform(9, 15)
    proj = Projector(g, 8, 8)
    cols = []
    for k in range(64):
        e = np.zeros(64)
        e[k] = 1.0
        cols.append(cpu(proj.forward(e.reshape(8, 8))).ravel())
    smax2 = float(np.linalg.svd(np.stack(cols, axis=1).astype(np.float64),
                                compute_uv=False)[0] ** 2)
    assert proj.norm_sq(30, 3) == proj.norm_sq(30, 3)
    ests = [proj.norm_sq(k, 0) for k in (1, 3, 10, 40, 200)]
    assert all(b >= a * (1 - 1e-6) for a, b in zip(ests, ests[1:]))
    assert ests[-1] <= smax2 * (1 + 1e-5)
    assert ests[-1] == pytest.approx(smax2, rel=1e-4)


# ---- estimators (test_estimators.py) ----------------------------------------

def test_svrg_has_zero_variance_at_the_snapshot(small):
    """At x = snapshot every subset's SVRG estimate is the full gradient."""
    _, proj, data, _ = small
    x = np.random.default_rng(2).random((16, 16))
    part = build_staggered_partition(12, 4)
    st = E.init_svrg_state(x, proj, data, refresh_period=4)
    full = E.full_gradient(x, proj, data)
    for i in range(4):
        assert rel(E.svrg_estimate(x, i, st, proj, data, part), full) <= 1e-5


def test_saga_with_the_current_table_is_the_full_gradient(small):
    """A table holding every subset's gradient at x: each SAGA estimate is
    the full gradient, and the running sum stays the table's sum."""
    _, proj, data, _ = small
    x = np.random.default_rng(3).random((16, 16))
    n = 4
    part = build_staggered_partition(12, n)
    grads = torch.stack([E._subset_gradient(x, i, proj, data, part) for i in range(n)])
    full = E.full_gradient(x, proj, data)
    for i in range(n):
        st = E.SagaState(grads.clone(), grads.sum(0))
        assert rel(E.saga_estimate_update(x, i, st, proj, data, part), full) <= 1e-5
        assert rel(st.running_sum, st.table.sum(0)) <= 1e-6


# ---- regularizers (test_regularizers.py) ------------------------------------

def test_tv_prox_vanishing_weight_is_the_identity():
    u = np.random.default_rng(1).standard_normal((4, 4))
    out, _ = tv_prox(u, 1.0, TvProxConfig(alpha=1e-30, inner_iterations=5, nonneg=False))
    assert np.allclose(cpu(out), u, atol=1e-6)
    out, _ = tv_prox(u, 1.0, TvProxConfig(alpha=1e-30, inner_iterations=5, nonneg=True))
    assert np.allclose(cpu(out), np.maximum(u, 0.0), atol=1e-6)


def _prox_objective(x, u, lam, nonneg):
    if nonneg and (x < 0).any():
        return math.inf
    dv = np.diff(x, axis=0)
    dh = np.diff(x, axis=1)
    tv = np.sum(np.sqrt(np.pad(dv, ((0, 1), (0, 0))) ** 2 + np.pad(dh, ((0, 0), (0, 1))) ** 2))
    return 0.5 * np.sum((x - u) ** 2) + lam * tv


def test_tv_prox_decreases_the_prox_objective():
    rng = np.random.default_rng(2)
    for trial in range(40):
        u = rng.standard_normal((6, 6))
        lam = float(rng.uniform(0.05, 2.0))
        nonneg = bool(trial % 2)
        if nonneg:
            u = np.abs(u)
        out, _ = tv_prox(u, 1.0, TvProxConfig(alpha=lam, inner_iterations=30, nonneg=nonneg))
        x = cpu(out).astype(np.float64)
        assert _prox_objective(x, u, lam, nonneg) <= _prox_objective(u, u, lam, nonneg) + 1e-5


def test_tv_prox_is_nonexpansive_at_high_accuracy():
    rng = np.random.default_rng(3)
    cfg = TvProxConfig(alpha=0.7, inner_iterations=2000, warm_start=False)
    for _ in range(5):
        u, v = rng.standard_normal((8, 8)), rng.standard_normal((8, 8))
        pu, _ = tv_prox(u, 1.0, cfg)
        pv, _ = tv_prox(v, 1.0, cfg)
        assert np.linalg.norm(cpu(pu) - cpu(pv)) <= np.linalg.norm(u - v) + 1e-5


def test_tv_prox_cold_calls_are_reproducible():
    u = np.random.default_rng(4).standard_normal((6, 6))
    cfg = TvProxConfig(alpha=0.9, inner_iterations=25, warm_start=False)
    a, _ = tv_prox(u, 1.0, cfg)
    b, _ = tv_prox(u, 1.0, cfg)
    assert torch.equal(a, b)


def test_tv_prox_warm_start_improves_accuracy(oracle):
    u = np.random.default_rng(8).standard_normal((5, 5))
    exact, _ = oracle.tv_prox(u, 1.0, 0.4, 20000, nonneg=False)
    cfg = TvProxConfig(alpha=0.4, inner_iterations=10, nonneg=False)
    state, errs = None, []
    for _ in range(30):
        out, state = tv_prox(u, 1.0, cfg, warm=state)
        errs.append(np.abs(cpu(out) - exact).max())
    assert errs[-1] < errs[0] / 10


# ---- solvers (test_solvers.py) ----------------------------------------------

def test_control_variate_stays_zero_without_prox_events(small):
    """p = 1e-12 never fires: h stays exactly zero and the trajectory is plain
    SGD with the same subset stream (test_solvers.py:37-62)."""
    problem, proj, data, lip = small
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=1e-12, estimator="sgd", n_subsets=4,
                       max_data_passes=1e9, seed=9)
    st = _init_state(cfg, problem, None)
    mirror = np.random.default_rng(np.random.SeedSequence(9).spawn(3)[0])
    x = torch.zeros((16, 16), device="cuda")
    for _ in range(50):
        proxskip_step(st, cfg, problem)
        i = int(mirror.integers(4))
        x = x - cfg.gamma * E.sgd_estimate(x, i, proj, data, st.partition)
    assert st.prox_calls == 0
    assert torch.count_nonzero(st.h) == 0
    assert rel(st.x, x) <= 1e-5


def test_full_gradient_at_p1_is_ista_bitwise(small):
    problem, _, _, lip = small
    cfg = SolverConfig(gamma=1.99 / lip, skip_probability=1.0, estimator="full",
                       max_data_passes=50, seed=1)
    a, b = run(cfg, problem), run_ista(cfg, problem)
    assert torch.equal(a.image, b.image)
    assert a.rows[-1][5] == b.rows[-1][5] == 50


@pytest.mark.parametrize("est", ["sgd", "saga"])
def test_single_subset_estimators_follow_the_ista_trajectory(small, est):
    """N = 1: the SGD / SAGA estimates are the full gradient, step by step and
    bit for bit (test_solvers.py:75-88)."""
    problem, _, _, lip = small
    a_cfg = SolverConfig(gamma=1.99 / lip, estimator="full", max_data_passes=1e9, seed=1)
    b_cfg = SolverConfig(gamma=1.99 / lip, estimator=est, n_subsets=1, max_data_passes=1e9,
                         seed=1)
    a, b = _init_state(a_cfg, problem, None), _init_state(b_cfg, problem, None)
    for _ in range(50):
        proxskip_step(a, a_cfg, problem)
        proxskip_step(b, b_cfg, problem)
        assert torch.equal(a.x, b.x)


def test_prox_call_count_is_binomial(small):
    problem, _, _, lip = small
    p = 0.3
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=p, estimator="sgd", n_subsets=5,
                       max_data_passes=400, seed=17)
    rec = run(cfg, problem)
    assert rec.iterations[-1] == 2000
    calls = rec.rows[-1][RUN_COLUMNS.index("prox_calls")]
    assert abs(calls - p * 2000) <= 3 * math.sqrt(2000 * p * (1 - p))


def test_infinite_tolerance_stops_at_the_initial_row(small):
    problem, _, _, lip = small
    cfg = SolverConfig(gamma=1.0 / lip, max_data_passes=100, tolerance=math.inf, seed=0)
    rec = run(cfg, problem, reference=np.ones((16, 16)))
    assert len(rec.rows) == 1 and rec.rows[0][0] == 0.0 and rec.iterations == [0]


def test_runs_are_deterministic_up_to_timing(small):
    problem, _, _, lip = small
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.4, estimator="svrg", n_subsets=4,
                       max_data_passes=30, seed=23)
    ref = np.ones((16, 16))
    a, b = run(cfg, problem, reference=ref), run(cfg, problem, reference=ref)
    assert torch.equal(a.image, b.image)
    t = RUN_COLUMNS.index("wall_seconds")
    for ra, rb in zip(a.rows, b.rows):
        assert [v for j, v in enumerate(ra) if j != t] == [v for j, v in enumerate(rb) if j != t]
    for name in ("data_passes", "wall_seconds", "prox_calls"):
        assert np.all(np.diff(a.column(name)) >= 0.0)


def test_no_rows_after_the_tolerance_is_met(small, tmp_path):
    problem, _, _, lip = small
    reference = run_pdhg_reference(problem, 20000)
    cfg = SolverConfig(gamma=1.99 / lip, max_data_passes=500, tolerance=1e-4, seed=0)
    rec = run(cfg, problem, reference=reference)
    below = rec.column("rel_err") < 1e-4
    assert below[-1] and not below[:-1].any()
    path = tmp_path / "rec.csv"
    rec.to_csv(path)
    lines = path.read_text().strip().splitlines()
    assert lines[0] == ",".join(RUN_COLUMNS)
    assert len(lines) == len(rec.rows) + 1


def test_data_pass_accounting(small):
    problem, _, _, lip = small
    rec = run(SolverConfig(gamma=1.0 / lip, max_data_passes=7, seed=0), problem)
    assert rec.rows[-1][0] == pytest.approx(7.0) and rec.iterations[-1] == 7
    rec = run(SolverConfig(gamma=1.0 / lip, estimator="sgd", n_subsets=4, max_data_passes=6,
                           seed=0), problem)
    assert rec.iterations[-1] == 24
    rec = run(SolverConfig(gamma=1.0 / lip, estimator="svrg", n_subsets=4, max_data_passes=10,
                           seed=0), problem)
    iters = rec.iterations[-1]
    assert rec.rows[-1][0] == pytest.approx(1.0 + iters * 0.5 + (iters - 1) // 4)


def test_objective_recorded_when_requested(small):
    problem, _, _, lip = small
    rec = run(SolverConfig(gamma=1.0 / lip, max_data_passes=3, seed=0), problem,
              record_objective=True)
    obj = rec.column("objective")
    assert np.all(np.isfinite(obj))
    assert obj[-1] == pytest.approx(composite_objective(rec.image, problem), rel=1e-5)
