"""Host-side logic (no GPU): the bit-exact subset / skip / refresh schedule,
pass accounting and log-row segmentation of the native run loop, the
geometry / partition contract and the synthetic-problem generators."""

import math

import numpy as np
import pytest

from paper_2602_09527_b200 import problems
from paper_2602_09527_b200.geometry import (ParallelGeometry, angle_sector,
                                            build_staggered_partition)
from paper_2602_09527_b200.solvers import (IterateState, SolverConfig, _draw_one, _plan_segment,
                                           default_gamma, fista_gamma, optimal_p)


def _state(config, n_angles):
    streams = np.random.SeedSequence(config.seed).spawn(3)
    part = (build_staggered_partition(n_angles, config.n_subsets)
            if config.estimator != "full" else None)
    st = IterateState(session=None, partition=part,
                      rng_subset=np.random.default_rng(streams[0]),
                      rng_theta=np.random.default_rng(streams[1]),
                      rng_refresh=np.random.default_rng(streams[2]))
    if config.estimator == "svrg":
        st.svrg_period = config.n_subsets
        st.data_passes = 1.0
    elif config.estimator == "lsvrg":
        st.svrg_probability = 1.0 / config.n_subsets
        st.data_passes = 1.0
    return st


def _simulate(config, n_angles):
    """The native run loop's host schedule, segment by segment."""
    st = _state(config, n_angles)
    subs, thetas, refr, rows, iters = [], [], [], [st.data_passes], [0]
    last_floor = math.floor(st.data_passes + 1e-12)
    k = 0
    while True:
        s, t, r, passes, exhausted = _plan_segment(st, config, last_floor)
        subs += list(s); thetas += list(t); refr += list(r)
        k += len(s)
        st.data_passes = passes
        if math.floor(passes + 1e-12) > last_floor or exhausted:
            last_floor = math.floor(passes + 1e-12)
            rows.append(passes)
            iters.append(k)
            if exhausted:
                break
    return np.array(subs), np.array(thetas), np.array(refr), rows, iters


@pytest.mark.parametrize("name,n,p,k,seed", [("c0", 10, 0.1, 500, 0), ("c1", 20, 0.05, 2000, 0),
                                             ("c2", 60, 0.05, 1800, 0), ("c3", 40, 0.1, 800, 0)])
def test_vectorised_schedule_equals_reference_draws(units, name, n, p, k, seed):
    est = "saga" if name == "c1" else "svrg"
    passes = {"c0": 150, "c1": 100, "c2": 90, "c3": 60}[name]
    cfg = SolverConfig(gamma=1.0, skip_probability=p, n_subsets=n, estimator=est,
                       max_data_passes=passes, seed=seed)
    subs, thetas, refr, rows, iters = _simulate(cfg, n * 30)
    assert len(subs) == k
    assert np.array_equal(subs, units[f"sched_{name}_subsets"])
    assert np.array_equal(thetas, units[f"sched_{name}_theta"])
    # SURVEY.md 8c seed-0 known answers
    known = {"c0": (46, 14, [8, 9, 0, 3, 7, 7, 2, 1, 9, 4]),
             "c1": (114, 15, [16, 18, 0, 6, 15, 14, 4, 2, 19, 8]),
             "c2": (93, 15, [48, 56, 0, 18, 45, 43, 12, 7, 58, 25]),
             "c3": (80, 14, [32, 37, 0, 12, 30, 28, 8, 5, 39, 16])}[name]
    assert int(thetas.sum()) == known[0]
    assert int(np.argmax(thetas)) == known[1]  # 0-based step index
    assert list(subs[:10]) == known[2]
    if est == "svrg":
        # snapshot refresh at the start of steps N, 2N, ... (estimators.py:156-157)
        assert list(np.nonzero(refr)[0]) == list(range(n, k, n))


def test_c0_row_schedule_matches_reference_run(c0_ref):
    cfg = SolverConfig(gamma=1.0, skip_probability=0.1, n_subsets=10, estimator="svrg",
                       max_data_passes=150.0, seed=0)
    subs, thetas, refr, rows, iters = _simulate(cfg, 180)
    assert np.array_equal(rows, c0_ref["c0_passes"])
    assert np.array_equal(iters, c0_ref["c0_iters"])


@pytest.mark.parametrize("est,p,passes,seed", [("full", 1.0, 20, 1), ("sgd", 0.4, 30, 17),
                                               ("saga", 0.4, 30, 3), ("svrg", 0.4, 30, 23),
                                               ("lsvrg", 0.5, 30, 4), ("svrg", 1.0, 15, 5)])
def test_small_run_rows_match_reference(small_runs, est, p, passes, seed):
    cfg = SolverConfig(gamma=1.0, skip_probability=p, n_subsets=5 if est != "full" else 1,
                       estimator=est, max_data_passes=passes, seed=seed)
    subs, thetas, refr, rows, iters = _simulate(cfg, 10)
    tag = f"small_{est}_p{p}_s{seed}"
    assert np.array_equal(rows, small_runs[tag + "_passes"])
    assert np.array_equal(iters, small_runs[tag + "_iters"])
    # prox calls at the final row
    assert int(np.count_nonzero(thetas)) == int(small_runs[tag + "_prox"][-1])


def test_lsvrg_refresh_stream(units):
    cfg = SolverConfig(gamma=1.0, skip_probability=0.5, n_subsets=5, estimator="lsvrg",
                       max_data_passes=1e9, seed=4)
    st = _state(cfg, 10)
    draws = [_draw_one(st, cfg)[2] for _ in range(400)]
    assert np.array_equal(draws, units["sched_lsvrg_refresh"])


def test_svrg_pass_accounting_formula():
    # reference tests/test_solvers.py:287-296: passes = 1 + iters*2/N + (iters-1)//N
    cfg = SolverConfig(gamma=1.0, estimator="svrg", n_subsets=5, max_data_passes=10, seed=0)
    subs, thetas, refr, rows, iters = _simulate(cfg, 10)
    assert rows[-1] == pytest.approx(1.0 + iters[-1] * (2.0 / 5.0) + (iters[-1] - 1) // 5)


def test_geometry_contract():
    g = ParallelGeometry.uniform(8, 11)
    assert g.angles[3] == 3 * math.pi / 8
    with pytest.raises(ValueError):
        ParallelGeometry((0.5, 0.2), 3)
    with pytest.raises(ValueError):
        ParallelGeometry((0.0, math.pi), 3)
    with pytest.raises(ValueError):
        ParallelGeometry((0.0,), 0)
    with pytest.raises(ValueError):
        ParallelGeometry((0.0,), 3, bin_spacing=0.0)
    with pytest.raises(ValueError):
        build_staggered_partition(5, 6)
    part = build_staggered_partition(10, 3)
    assert part.subsets == ((0, 3, 6, 9), (1, 4, 7), (2, 5, 8))


def test_angle_sectors_partition_every_subset():
    for A, G in ((1800, 8), (720, 4), (180, 2), (7, 3)):
        sectors = [angle_sector(A, r, G) for r in range(G)]
        assert sectors[0][0] == 0 and sectors[-1][1] == A
        assert all(a[1] == b[0] for a, b in zip(sectors, sectors[1:]))
    with pytest.raises(ValueError):
        angle_sector(10, 2, 2)


def test_step_size_rules():
    assert default_gamma("full", 2.0) == pytest.approx(1.99 / 2.0)
    assert default_gamma("saga", 2.0) == pytest.approx(1.0 / 6.0)
    assert default_gamma("svrg", 2.0) == 0.5
    assert fista_gamma(2.0) == 0.5
    assert optimal_p(0.01, 1.0) == pytest.approx(0.1)
    with pytest.raises(ValueError):
        default_gamma("sarah", 1.0)


def test_config_validation():
    for kw in ({"gamma": 0.0}, {"gamma": 1.0, "skip_probability": 0.0},
               {"gamma": 1.0, "skip_probability": 1.2}, {"gamma": 1.0, "estimator": "sarah"},
               {"gamma": 1.0, "n_subsets": 0}, {"gamma": 1.0, "max_data_passes": 0.0}):
        with pytest.raises(ValueError):
            SolverConfig(**kw)


def test_phantom_generators_deterministic():
    a = problems.ellipse_phantom(64, 10, 0)
    b = problems.ellipse_phantom(64, 10, 0)
    assert np.array_equal(a, b) and a.max() > 0.1 and a.min() >= 0.0
    v = problems.ellipsoid_phantom(32, 5, 0)
    assert v.shape == (32, 32, 32) and v.max() > 0.1
    clean = np.abs(np.random.default_rng(0).standard_normal((4, 9)))
    noisy = problems.add_noise(clean, "poisson-like", 1)
    assert noisy.shape == clean.shape and not np.array_equal(noisy, clean)
    cfg = problems.CONFIGS["c2"]
    assert cfg.max_data_passes == 90.0 and cfg.n_subsets == 60
