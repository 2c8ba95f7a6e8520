"""Parity at the benchmarked sizes (BASELINE configs 2 and 3) against the
pinned float64 oracle (oracle/, pinned to the reference's own outputs in
tests/test_oracle.py; the reference itself cannot run these sizes: its
explicit CSR would need ~215 GB at config 2).

* the full 1800-angle forward and adjoint at 2048^2 (the snapshot's
  angle-grouped launches) and subsets across the partition: rel-L2 <= 1e-5;
* config 2 for two epochs (2048^2, 1800x2900, SVRG N=60, p=0.05, FGP-100):
  the segment contains the initial snapshot, a refresh at step 60, the
  post-refresh step (whose subset projection is skipped because x == x_snap)
  and several FGP-100 calls; iteration / prox / row schedule bit-exact,
  final iterate and objective rel-L2 <= 1e-4 (north_star);
* config 3's geometry and law on a 64-plane slab (256^2 x 64, 360x384,
  SVRG N=40, p=0.1, 3D FGP-100) for 1.25 epochs (a refresh included).

Reference call sites: pkg/src/proxtomo/solvers.py:327-336 (run),
estimators.py:40-48,133-146 (full gradient, SVRG estimate),
projector.py:114-140 (forward / adjoint), regularizers.py:90-133 (FGP)."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from paper_2602_09527_b200 import (ParallelGeometry, Projector, SolverConfig, TomoProblem,
                                   TvProxConfig, composite_objective, default_gamma, problems,
                                   run)

pytestmark = pytest.mark.gpu
TOL_PROJ = 1e-5
TOL_RUN = 1e-4


def cpu(t):
    return t.detach().double().cpu().numpy()


@pytest.fixture(scope="module")
def fast_oracle():
    import oracle as O
    O.set_mode("fast")
    yield O
    O.set_mode("exact")


@pytest.fixture(scope="module")
def c2_problem(fast_oracle):
    """Config 2's b from the float64 oracle (phantom law, Poisson-like noise)."""
    O = fast_oracle
    cfg = problems.CONFIGS["c2"]
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    x_true = problems.phantom_for(cfg)
    b = problems.add_noise(O.forward_project(x_true, g), cfg.noise, cfg.noise_seed)
    return cfg, g, x_true, b


def test_full_forward_adjoint_2048(c2_problem, fast_oracle):
    """All 1800 angles at once (the SVRG snapshot's launch, up to 16 angle
    groups) and subsets from across the partition, against float64."""
    O = fast_oracle
    cfg, g, x_true, b = c2_problem
    proj = Projector(g, cfg.size, cfg.size)
    rng = np.random.default_rng(11)
    x = x_true + 0.1 * rng.random(x_true.shape)
    y = proj.forward(x)
    y_ref = O.forward_project(x, g)
    assert rel_l2(cpu(y), y_ref) <= TOL_PROJ
    r = b - y_ref
    a = proj.adjoint(r)
    assert rel_l2(cpu(a), O.back_project(r, g, (cfg.size, cfg.size))) <= TOL_PROJ
    for k in (1, 17, 29, 44):
        sub = tuple(range(k, cfg.n_angles, cfg.n_subsets))
        ys = proj.forward(x, sub)
        assert rel_l2(cpu(ys), y_ref[list(sub)]) <= TOL_PROJ
        a_s = proj.adjoint(r[list(sub)], sub)
        assert rel_l2(cpu(a_s), O.back_project(r[list(sub)], g, (cfg.size, cfg.size), sub)) \
            <= TOL_PROJ


def test_config2_two_epochs_match_oracle(c2_problem, fast_oracle):
    O = fast_oracle
    from oracle import solver as S
    cfg, g, _, b = c2_problem
    proj = Projector(g, cfg.size, cfg.size)
    b_dev = torch.tensor(b, device="cuda", dtype=torch.float32)
    alpha = problems.alpha_from_backprojection(float(proj.adjoint(b_dev).abs().max()),
                                               cfg.n_pixels)
    lip = proj.norm_sq(cfg.power_iterations, cfg.power_seed)
    gamma = default_gamma(cfg.estimator, lip)
    passes = 6.0  # 2 SVRG epochs: init snapshot + 60 steps + refresh + 60 steps
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=passes, seed=cfg.solver_seed)
    tv = TvProxConfig(alpha=alpha, inner_iterations=cfg.fgp_inner)
    problem = TomoProblem(proj, b_dev, tv=tv)
    rec = run(scfg, problem)
    ref = S.run_proxskip(O.OracleProjector(g, cfg.size, cfg.size), b, gamma=gamma, p=cfg.p,
                         estimator=cfg.estimator, n_subsets=cfg.n_subsets,
                         max_data_passes=passes, seed=cfg.solver_seed, tv_alpha=alpha,
                         tv_inner=cfg.fgp_inner)
    assert ref.k == 120 and rec.iterations == ref.iterations
    assert list(rec.column("prox_calls")) == [row[2] for row in ref.rows]
    assert ref.prox_calls >= 2  # FGP-100 calls inside the compared segment
    assert np.array_equal(rec.column("data_passes"), [row[0] for row in ref.rows])
    assert rel_l2(cpu(rec.image), ref.image) <= TOL_RUN
    obj = composite_objective(rec.image, problem)
    obj_ref = S.objective(O.OracleProjector(g, cfg.size, cfg.size), b, ref.image, alpha)
    assert obj == pytest.approx(obj_ref, rel=TOL_RUN)


def test_config3_slab_matches_oracle(fast_oracle):
    """Config 3's geometry (360 angles x 384 bins), ellipsoid law and solver
    (SVRG N=40, p=0.1, isotropic 3D FGP-100) on 64 planes of the 256^3
    volume, 50 iterations (a refresh at step 40 and its post-refresh step)."""
    O = fast_oracle
    from oracle import solver as S
    cfg = problems.CONFIGS["c3"]
    Z = 64
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    vol = np.ascontiguousarray(problems.phantom_for(cfg)[96:96 + Z]).astype(np.float64)
    b = problems.add_noise(O.forward_project(vol, g), cfg.noise, cfg.noise_seed)  # (Z, A, B)
    b_dev = torch.tensor(b.transpose(1, 0, 2), device="cuda",
                         dtype=torch.float32).contiguous()  # device layout (A, Z, B)
    proj = Projector(g, cfg.size, cfg.size, n_slices=Z)
    alpha = problems.alpha_from_backprojection(float(proj.adjoint(b_dev).abs().max()),
                                               cfg.size * cfg.size * Z)
    # raise TV so the 3D prox visibly moves the iterate
    alpha *= 20.0
    lip = proj.norm_sq(cfg.power_iterations, cfg.power_seed)
    gamma = default_gamma(cfg.estimator, lip)
    passes = 4.5  # init + 40 steps + refresh + 10 steps
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=passes, seed=cfg.solver_seed)
    rec = run(scfg, TomoProblem(proj, b_dev, tv=TvProxConfig(alpha=alpha,
                                                               inner_iterations=cfg.fgp_inner)))
    oproj = O.OracleProjector(g, cfg.size, cfg.size, n_slices=Z)
    b_am = np.ascontiguousarray(b.transpose(1, 0, 2))
    ref = S.run_proxskip(_SliceMajor(oproj), b_am, gamma=gamma, p=cfg.p, estimator=cfg.estimator,
                         n_subsets=cfg.n_subsets, max_data_passes=passes, seed=cfg.solver_seed,
                         tv_alpha=alpha, tv_inner=cfg.fgp_inner)
    assert ref.k == 50 and rec.iterations == ref.iterations
    assert list(rec.column("prox_calls")) == [row[2] for row in ref.rows]
    assert ref.prox_calls >= 2
    assert rel_l2(cpu(rec.image), ref.image) <= TOL_RUN


class _SliceMajor:
    """The oracle's slice-stacked projector with the subset index on axis 1
    ((Z, n_sel, B) sinograms), as run_proxskip indexes data[list(s)] on axis 0:
    present the data / projections angle-major to it."""

    def __init__(self, oproj):
        self._p = oproj
        self.geometry = oproj.geometry
        self.shape = oproj.shape

    def forward(self, image, subset=None):
        return self._p.forward(image, subset).transpose(1, 0, 2)

    def adjoint(self, sino, subset=None):
        return self._p.adjoint(np.ascontiguousarray(np.asarray(sino).transpose(1, 0, 2)), subset)
