"""The reference-side binding (INTEGRATION.md Option B) driven by the
reference's own loop: ``B200Projector`` duck-types proxtomo's ``Projector``
(pkg/src/proxtomo/projector.py:143-167; any such object works,
pkg/tests/test_estimators.py:69-82) and is handed to the float64 restatement
of ``run()`` (oracle/solver.py, pinned bit-for-bit to the reference's runs in
tests/test_oracle.py).  Only the CSR SpMVs move to the GPU; the estimator,
ProxSkip step and FGP stay the reference's float64 numpy/C."""

import numpy as np
import pytest

from conftest import rel_l2
from paper_2602_09527_b200 import ParallelGeometry, problems
from paper_2602_09527_b200.reference_binding import B200Projector

pytestmark = pytest.mark.gpu


def test_binding_projector_matches_reference_goldens(units, oracle):
    g = ParallelGeometry.uniform(30, 45)
    proj = B200Projector(g, 32, 28)
    oproj = oracle.OracleProjector(g, 32, 28)
    rng = np.random.default_rng(4)
    x = rng.random((28, 32))
    sub = (1, 4, 9, 20)
    assert rel_l2(proj.forward(x), oproj.forward(x)) <= 1e-5
    assert rel_l2(proj.forward(x, sub), oproj.forward(x, sub)) <= 1e-5
    y = rng.standard_normal((4, 45))
    assert rel_l2(proj.adjoint(y, sub), oproj.adjoint(y, sub)) <= 1e-5
    assert proj.shape == (28, 32)
    with pytest.raises(ValueError):
        proj.forward(np.zeros((3, 3)))
    with pytest.raises(ValueError):
        proj.adjoint(np.zeros((5, 45)), sub)
    with pytest.raises(ValueError):
        proj.forward(x, (30,))
    assert proj.norm_sq(20, 0) == pytest.approx(oproj.norm_sq(20, 0), rel=1e-5)


def test_reference_loop_with_binding_reproduces_config0(c0_ref, oracle):
    """BASELINE config 0 whole (128^2, 180x192, SVRG N=10, p=0.1, FGP 50,
    500 iterations) through the reference's loop with the B200 projector:
    final iterate and objective within 1e-4 of the reference's own run,
    prox-call and row schedule identical."""
    from oracle import solver as S
    cfg = problems.CONFIGS["c0"]
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = B200Projector(g, cfg.size, cfg.size)
    r = S.run_proxskip(proj, c0_ref["c0_b"], gamma=float(c0_ref["c0_gamma"]), p=cfg.p,
                       estimator=cfg.estimator, n_subsets=cfg.n_subsets,
                       max_data_passes=cfg.max_data_passes, seed=cfg.solver_seed,
                       tv_alpha=float(c0_ref["c0_alpha"]), tv_inner=cfg.fgp_inner,
                       record_objective=True)
    assert rel_l2(r.image, c0_ref["c0_image"]) <= 1e-4
    assert r.iterations == list(c0_ref["c0_iters"])
    assert [row[2] for row in r.rows] == list(c0_ref["c0_prox"])
    obj = np.array([row[3] for row in r.rows])
    assert np.allclose(obj, c0_ref["c0_obj"], rtol=1e-4)
