"""Error behaviour of the reference-facing API: every invalid argument the
reference's own unit tests reject (pkg/tests/test_geometry.py:40-63,
test_estimators.py:101-104,212-222, test_metrics.py:19-31,96-115,
test_regularizers.py:112,286-289, test_solvers.py:185-188,221-272,
test_projector.py:116-129,181) raises the same exception type here.  The
host-side checks run without a GPU; the ones that need a device plan are
marked."""
import math

import numpy as np
import pytest
import torch

from paper_2602_09527_b200 import (ParallelGeometry, SolverConfig, SubsetPartition, TvProxConfig,
                                   build_staggered_partition, default_gamma, optimal_p)
from paper_2602_09527_b200.estimators import (SvrgState, refresh_policy, sgd_estimate,
                                              svrg_estimate)
from paper_2602_09527_b200.metrics import StoppingRule, psnr


@pytest.mark.parametrize("args,kw", [
    (((), 5), {}),
    (((0.3, 0.2), 5), {}),
    (((0.0, math.pi), 5), {}),
    (((0.0,), 0), {}),
    (((0.0,), 5), {"bin_spacing": 0.0}),
    (((0.0,), 5), {"pixel_size": -1.0}),
])
def test_geometry_rejects(args, kw):
    with pytest.raises(ValueError):
        ParallelGeometry(*args, **kw)


@pytest.mark.parametrize("bad", [0, 8, -1])
def test_partition_size_rejected(bad):
    with pytest.raises(ValueError):
        build_staggered_partition(7, bad)


def test_partition_must_cover_exactly_once():
    with pytest.raises(ValueError):
        SubsetPartition(4, ((0, 1), (3,)))
    with pytest.raises(ValueError):
        SubsetPartition(3, ((0, 1), (1, 2)))


def test_estimator_argument_checks():
    part = build_staggered_partition(6, 3)
    x = torch.zeros((4, 4))
    # the subset index is checked before any projection
    for bad in (3, -1):
        with pytest.raises(ValueError):
            sgd_estimate(x, bad, None, None, part)
    with pytest.raises(ValueError):
        SvrgState(snapshot=x, full_grad=x)
    with pytest.raises(ValueError):
        SvrgState(snapshot=x, full_grad=x, refresh_period=3, refresh_probability=0.1)
    stale = SvrgState(snapshot=x, full_grad=x, refresh_period=3)
    stale.iterations_since_refresh = 4
    with pytest.raises(ValueError, match="stale"):
        svrg_estimate(x, 0, stale, None, None, part)
    with pytest.raises(ValueError):
        refresh_policy(SvrgState(snapshot=x, full_grad=x, refresh_probability=0.5))


@pytest.mark.parametrize("kw", [{"tolerance": 1e-5}, {"max_data_passes": math.inf},
                                {"max_data_passes": -1.0}, {"time_budget": 0.0}])
def test_stopping_rule_rejects(kw):
    with pytest.raises(ValueError):
        StoppingRule(**kw)


def test_metric_argument_checks():
    with pytest.raises(ValueError):
        psnr(np.ones((3, 3)), np.ones((3, 3)), 0.0)


@pytest.mark.parametrize("kw", [{"alpha": 0.0}, {"alpha": 1.0, "inner_iterations": 0}])
def test_tv_config_rejects(kw):
    with pytest.raises(ValueError):
        TvProxConfig(**kw)


def test_step_size_helpers_reject():
    for mu, lip in ((2.0, 1.0), (0.0, 1.0), (1.0, -1.0)):
        with pytest.raises(ValueError):
            optimal_p(mu, lip)
    with pytest.raises(ValueError):
        default_gamma("full", 0.0)


@pytest.mark.parametrize("kw", [{"gamma": 0.0}, {"gamma": 1.0, "skip_probability": 0.0},
                                {"gamma": 1.0, "skip_probability": 1.2},
                                {"gamma": 1.0, "estimator": "sarah"},
                                {"gamma": 1.0, "n_subsets": 0},
                                {"gamma": 1.0, "max_data_passes": 0.0}])
def test_solver_config_rejects(kw):
    with pytest.raises(ValueError):
        SolverConfig(**kw)


@pytest.mark.gpu
def test_device_side_argument_checks():
    """Checks that need a device plan: projector subsets and shapes, the
    operator-norm iteration count, the TV step, the problem's data shape,
    metrics of a zero reference / mismatched shapes."""
    from paper_2602_09527_b200 import (Projector, TomoProblem, back_project, forward_project,
                                       operator_norm_sq, tv_prox)
    from paper_2602_09527_b200.metrics import relative_error_sq, ssim
    g = ParallelGeometry.uniform(4, 9)
    with pytest.raises(ValueError):
        forward_project(np.zeros((4, 4)), g, subset=(0, 5))
    with pytest.raises(ValueError):
        back_project(np.zeros((2, 9)), g, (4, 4), subset=(-1, 0))
    with pytest.raises(ValueError):
        back_project(np.zeros((3, 9)), g, (4, 4), subset=(0, 1))
    with pytest.raises(ValueError):
        forward_project(np.zeros(16), g)
    with pytest.raises(ValueError):
        operator_norm_sq(g, 5, 5, iterations=0)
    with pytest.raises(ValueError):
        tv_prox(np.zeros((3, 3)), 0.0, TvProxConfig(alpha=1.0))
    with pytest.raises(ValueError):
        TomoProblem(Projector(g, 4, 4), np.zeros((3, 3)))
    with pytest.raises(ValueError):
        relative_error_sq(np.ones((3, 3)), np.zeros((3, 3)))
    with pytest.raises(ValueError):
        ssim(np.ones((4, 4)), np.ones((5, 5)))
