"""End-to-end parity of the native ProxSkip executor (csrc/session.cu).

* subset / skip / refresh sequences: bit-exact (prox-call counts, rows,
  iterations identical to the reference's);
* final iterate and objective after K epochs: relative L2 <= 1e-4 against
  the reference's own runs (tests/golden) -- config 0 whole, and the 16^2
  problem for every estimator."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from paper_2602_09527_b200 import (DivergenceError, ParallelGeometry, Projector, SolverConfig,
                                   TomoProblem, TvProxConfig, composite_objective, default_gamma,
                                   proxskip_step, run, run_fista, run_ista)
from paper_2602_09527_b200 import estimators as E
from paper_2602_09527_b200 import problems
from paper_2602_09527_b200.solvers import _init_state

pytestmark = pytest.mark.gpu
TOL = 1e-4


def cpu(t):
    return t.detach().double().cpu().numpy()


def small_problem(small_runs):
    g = ParallelGeometry.uniform(10, 23)
    proj = Projector(g, 16, 16)
    tv = TvProxConfig(alpha=0.5, inner_iterations=10)
    return TomoProblem(proj, small_runs["small_data"], tv=tv), float(small_runs["small_L"])


@pytest.mark.parametrize("est,p,passes,seed", [("full", 1.0, 20, 1), ("sgd", 0.4, 30, 17),
                                               ("saga", 0.4, 30, 3), ("svrg", 0.4, 30, 23),
                                               ("lsvrg", 0.5, 30, 4), ("svrg", 1.0, 15, 5)])
def test_small_runs_match_reference(small_runs, est, p, passes, seed):
    problem, lip = small_problem(small_runs)
    cfg = SolverConfig(gamma=default_gamma(est, lip), skip_probability=p,
                       n_subsets=5 if est != "full" else 1, estimator=est,
                       max_data_passes=passes, seed=seed)
    rec = run(cfg, problem, record_objective=True)
    tag = f"small_{est}_p{p}_s{seed}"
    assert rel_l2(cpu(rec.image), small_runs[tag + "_image"]) <= TOL
    assert np.array_equal(rec.column("data_passes"), small_runs[tag + "_passes"])
    assert np.array_equal(rec.column("prox_calls"), small_runs[tag + "_prox"])
    assert rec.iterations == list(small_runs[tag + "_iters"])
    obj = rec.column("objective")
    assert np.allclose(obj, small_runs[tag + "_obj"], rtol=TOL)


def test_config0_whole_run_matches_reference(c0_ref):
    """BASELINE config 0: 128^2, 180x192, SVRG N=10, p=0.1, FGP 50, 50 epochs."""
    cfg = problems.CONFIGS["c0"]
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = Projector(g, cfg.size, cfg.size)
    tv = TvProxConfig(alpha=float(c0_ref["c0_alpha"]), inner_iterations=cfg.fgp_inner)
    problem = TomoProblem(proj, c0_ref["c0_b"], tv=tv)
    scfg = SolverConfig(gamma=float(c0_ref["c0_gamma"]), skip_probability=cfg.p,
                        n_subsets=cfg.n_subsets, estimator=cfg.estimator,
                        max_data_passes=cfg.max_data_passes, seed=cfg.solver_seed)
    rec = run(scfg, problem, record_objective=True)
    assert rel_l2(cpu(rec.image), c0_ref["c0_image"]) <= TOL
    assert np.array_equal(rec.column("data_passes"), c0_ref["c0_passes"])
    assert np.array_equal(rec.column("prox_calls"), c0_ref["c0_prox"])
    assert rec.iterations == list(c0_ref["c0_iters"])
    assert np.allclose(rec.column("objective"), c0_ref["c0_obj"], rtol=TOL)
    walls = rec.column("wall_seconds")
    assert np.all(np.diff(walls) >= 0) and walls[-1] > 0


def test_config0_setup_constants_match_reference(c0_ref):
    """L (50 power iterations, seed 0) and alpha from the device operator."""
    cfg = problems.CONFIGS["c0"]
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = Projector(g, cfg.size, cfg.size)
    assert proj.norm_sq(50, 0) == pytest.approx(float(c0_ref["c0_L"]), rel=1e-5)
    atb = proj.adjoint(c0_ref["c0_b"])
    alpha = problems.alpha_from_backprojection(float(atb.abs().max()), cfg.n_pixels)
    assert alpha == pytest.approx(float(c0_ref["c0_alpha"]), rel=1e-5)


def test_proxskip_step_api_matches_run(small_runs):
    problem, lip = small_problem(small_runs)
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.4, n_subsets=5, estimator="svrg",
                       max_data_passes=1e9, seed=23)
    st = _init_state(cfg, problem, None)
    for _ in range(40):
        proxskip_step(st, cfg, problem)
    cfg2 = SolverConfig(gamma=1.0 / lip, skip_probability=0.4, n_subsets=5, estimator="svrg",
                        max_data_passes=st.data_passes, seed=23)
    rec = run(cfg2, problem)
    assert rec.iterations[-1] == st.k == 40
    assert torch.equal(rec.image, st.x)


def test_estimator_api_against_oracle(oracle):
    g = ParallelGeometry.uniform(6, 7)
    proj = Projector(g, 4, 4)
    oproj = oracle.OracleProjector(g, 4, 4)
    rng = np.random.default_rng(0)
    x, data = rng.standard_normal((4, 4)), rng.standard_normal((6, 7))
    full_ref = oproj.adjoint(oproj.forward(x) - data)
    assert rel_l2(cpu(E.full_gradient(x, proj, data)), full_ref) <= 1e-5
    from paper_2602_09527_b200 import build_staggered_partition
    for n in (2, 3, 6):
        part = build_staggered_partition(6, n)
        sgd = np.mean([cpu(E.sgd_estimate(x, i, proj, data, part)) for i in range(n)], axis=0)
        assert rel_l2(sgd, full_ref) <= 1e-5
        st = E.init_svrg_state(rng.standard_normal((4, 4)), proj, data, refresh_period=n)
        svrg = np.mean([cpu(E.svrg_estimate(x, i, st, proj, data, part)) for i in range(n)], axis=0)
        assert rel_l2(svrg, full_ref) <= 1e-4
        table = rng.standard_normal((n, 4, 4))
        saga = np.mean([cpu(E.saga_estimate_update(
            x, i, E.SagaState(torch.tensor(table, device="cuda", dtype=torch.float32),
                              torch.tensor(table.sum(0), device="cuda", dtype=torch.float32)),
            proj, data, part)) for i in range(n)], axis=0)
        assert rel_l2(saga, full_ref) <= 1e-4


def test_divergence_raises_with_partial_record():
    g = ParallelGeometry((0.0,), 1, bin_spacing=1.0, pixel_size=1.0)
    problem = TomoProblem(Projector(g, 1, 1), np.array([[1.0]]))
    cfg = SolverConfig(gamma=1e6, max_data_passes=2000, seed=0)
    with pytest.raises(DivergenceError) as info:
        run(cfg, problem)
    assert info.value.gamma == 1e6
    assert info.value.iteration > 0
    assert info.value.record is not None and len(info.value.record.rows) >= 1


def test_scalar_contraction_any_p():
    """f = x^2/2, g = 0: x <- (1 - gamma) x exactly (reference test_solvers.py:23-34)."""
    g = ParallelGeometry((0.0,), 1, bin_spacing=1.0, pixel_size=1.0)
    problem = TomoProblem(Projector(g, 1, 1), np.array([[0.0]]))
    for p in (1.0, 0.4, 0.05):
        cfg = SolverConfig(gamma=0.3, skip_probability=p, max_data_passes=1e9, seed=5)
        st = _init_state(cfg, problem, np.array([[2.0]]))
        value = 2.0
        for _ in range(40):
            proxskip_step(st, cfg, problem)
            value *= 0.7
            assert float(st.x[0, 0]) == pytest.approx(value, rel=1e-5)


@pytest.fixture(scope="module")
def fista_ref():
    import os
    from conftest import GOLDEN
    return np.load(os.path.join(GOLDEN, "reference_fista.npz"))


@pytest.mark.parametrize("name,tag", [("fista", "tv"), ("fista", "plain"), ("ista", "tv"),
                                      ("ista", "plain")])
def test_fista_ista_match_reference(small_runs, fista_ref, name, tag):
    """Native FISTA (momentum kernel, t_k in float64 on the host side of the
    session) and ISTA (ProxSkip full/p=1) vs the reference's run_fista /
    run_ista (solvers.py:339-392): 40 passes, rows and objective."""
    problem, lip = small_problem(small_runs)
    if tag == "plain":
        problem = TomoProblem(problem.projector, small_runs["small_data"])
    fn = run_fista if name == "fista" else run_ista
    # estimator / skipping fields are ignored by both (solvers.py:346-350)
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.3, n_subsets=5, estimator="svrg",
                       max_data_passes=40, seed=0)
    rec = fn(cfg, problem, record_objective=True)
    key = f"small_{name}_{tag}"
    assert rel_l2(cpu(rec.image), fista_ref[key + "_image"]) <= TOL
    assert rec.iterations == list(fista_ref[key + "_iters"])
    assert np.array_equal(rec.column("prox_calls"), fista_ref[key + "_prox"])
    assert np.allclose(rec.column("objective"), fista_ref[key + "_obj"], rtol=TOL)


def test_fista_config0_matches_reference(c0_ref, fista_ref):
    """20 FISTA passes of BASELINE config 0 (the config-4 f* solver's path)."""
    cfg = problems.CONFIGS["c0"]
    proj = Projector(ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins), cfg.size, cfg.size)
    problem = TomoProblem(proj, c0_ref["c0_b"], tv=TvProxConfig(alpha=float(c0_ref["c0_alpha"]),
                                                                 inner_iterations=cfg.fgp_inner))
    rec = run_fista(SolverConfig(gamma=1.0 / float(c0_ref["c0_L"]), max_data_passes=20),
                    problem, record_objective=True)
    assert rel_l2(cpu(rec.image), fista_ref["c0_fista_image"]) <= TOL
    assert np.allclose(rec.column("objective"), fista_ref["c0_fista_obj"], rtol=TOL)
    assert rec.iterations == list(fista_ref["c0_fista_iters"])


def test_fista_one_pass_equals_ista(small_runs):
    problem, lip = small_problem(small_runs)
    cfg = SolverConfig(gamma=1.0 / lip, max_data_passes=1, seed=0)
    assert torch.equal(run_fista(cfg, problem).image, run_ista(cfg, problem).image)


def test_fista_angle_sectors_match_single_device(small_runs):
    """FISTA on emulated angle sectors (partial gradients summed, then the
    shared epilogue / prox / momentum): the single-device trajectory."""
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200.solvers import _full_gradient_config, _init_state, _plan_segment
    problem, lip = small_problem(small_runs)
    cfg = _full_gradient_config(SolverConfig(gamma=1.0 / lip, max_data_passes=1e9))
    outs = []
    for w in (1, 3):
        st = _init_state(cfg, TomoProblem(problem.projector, small_runs["small_data"],
                                          tv=problem.tv), None, kind="fista")
        if w > 1:
            D.emulate_sectors(st.session, w)
        subs, th, rf, _, _ = _plan_segment(st, cfg, 1 << 40, max_steps=25)
        st.session.run(subs, th, rf, 0)
        outs.append(cpu(st.x))
    assert rel_l2(outs[1], outs[0]) <= 1e-5


def test_objective(small_runs):
    problem, lip = small_problem(small_runs)
    x = np.random.default_rng(1).random((16, 16))
    from oracle.solver import objective
    import oracle as O
    oproj = O.OracleProjector(ParallelGeometry.uniform(10, 23), 16, 16)
    want = objective(oproj, small_runs["small_data"], x, 0.5)
    assert composite_objective(x, problem) == pytest.approx(want, rel=1e-5)


@pytest.mark.parametrize("est,world", [("svrg", 2), ("svrg", 3), ("saga", 4), ("full", 2),
                                       ("sgd", 8)])
def test_angle_sector_decomposition_matches_single_rank(est, world):
    """The multi-GPU data path (each rank's own angle sector of subset i, the
    partial A_i^T r summed -- ncclAllReduce on real ranks -- then the shared
    epilogue and prox) emulated on one device: same trajectory as one rank,
    up to float32 summation order."""
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200 import problems
    from paper_2602_09527_b200.solvers import _init_state, _plan_segment
    g = ParallelGeometry.uniform(120, 97)
    proj = Projector(g, 64, 64)
    x_true = problems.ellipse_phantom(64, 6, 2)
    data = cpu(proj.forward(x_true)) + 0.01 * np.random.default_rng(0).standard_normal((120, 97))
    tv = TvProxConfig(alpha=0.2, inner_iterations=10)
    lip = proj.norm_sq(30, 0)
    outs = []
    for w in (1, world):
        problem = TomoProblem(proj, data, tv=tv)
        cfg = SolverConfig(gamma=default_gamma(est, lip), skip_probability=0.3,
                           n_subsets=6 if est != "full" else 1, estimator=est,
                           max_data_passes=1e9, seed=3)
        st = _init_state(cfg, problem, None)
        if w > 1:
            D.emulate_sectors(st.session, w)
            if est in ("svrg", "lsvrg"):
                st.session.init()  # snapshot gradient through the sectors
        subs, th, rf, passes, _ = _plan_segment(st, cfg, 1 << 40, max_steps=40)
        st.session.run(subs, th, rf, 0)
        outs.append(cpu(st.x))
    assert rel_l2(outs[1], outs[0]) <= 1e-5


def test_config1_whole_run_matches_reference(oracle):
    """BASELINE config 1 whole: 512^2, 720x768, SAGA N=20 (20x512^2 table),
    p=0.05, FGP 100, 100 epochs = 2000 iterations, against the reference's
    own run (tests/golden/reference_c1.npz; b regenerated with the pinned
    oracle): final image, row schedule, prox calls and the objective of
    every row."""
    import os
    from conftest import GOLDEN
    from test_oracle import config1_problem
    c1 = np.load(os.path.join(GOLDEN, "reference_c1.npz"))
    cfg, g, b = config1_problem(oracle)
    proj = Projector(g, cfg.size, cfg.size)
    tv = TvProxConfig(alpha=float(c1["c1_alpha"]), inner_iterations=cfg.fgp_inner)
    problem = TomoProblem(proj, b, tv=tv)
    scfg = SolverConfig(gamma=float(c1["c1_gamma"]), skip_probability=cfg.p,
                        n_subsets=cfg.n_subsets, estimator=cfg.estimator,
                        max_data_passes=cfg.max_data_passes, seed=cfg.solver_seed)
    rec = run(scfg, problem, record_objective="c1_obj" in c1.files)
    assert rel_l2(cpu(rec.image), c1["c1_image"]) <= TOL
    assert np.array_equal(rec.column("data_passes"), c1["c1_passes"])
    assert np.array_equal(rec.column("prox_calls"), c1["c1_prox"])
    assert rec.iterations == list(c1["c1_iters"])
    if "c1_obj" in c1.files:  # the objective at each of the 101 rows
        assert np.allclose(rec.column("objective"), c1["c1_obj"], rtol=TOL)
    assert proj.norm_sq(50, 0) == pytest.approx(float(c1["c1_L"]), rel=1e-5)


def test_nccl_data_path_on_one_rank_is_bitwise_identical(small_runs):
    """The multi-GPU data path through a real (one-rank) NCCL communicator:
    dlopen of torch's libnccl, unique-id exchange over torch.distributed,
    partial gradient -> ncclAllReduce -> separate epilogue kernel.  With one
    rank it must reproduce the fused single-GPU path bit for bit."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        problem, lip = small_problem(small_runs)
        cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.4, n_subsets=5,
                           estimator="svrg", max_data_passes=30, seed=23)
        a = run(cfg, problem)
        b = run(cfg, TomoProblem(problem.projector, small_runs["small_data"], tv=problem.tv),
                data_parallel=True)
        assert torch.equal(a.image, b.image)
        assert a.iterations == b.iterations
    finally:
        dist.destroy_process_group()


def test_pdhg_reference_matches_reference():
    """Device PDHG (pdhg.cu + projector) vs the reference's own PDHG runs."""
    import os
    from conftest import GOLDEN
    from paper_2602_09527_b200 import run_pdhg_reference
    f = np.load(os.path.join(GOLDEN, "reference_pdhg.npz"))
    proj = Projector(ParallelGeometry.uniform(10, 23), 16, 16)
    x, snap = run_pdhg_reference(TomoProblem(proj, f["pdhg_data"], tv=TvProxConfig(alpha=0.5)),
                                 300, snapshot_at=40)
    assert rel_l2(cpu(x), f["pdhg_tv_x"]) <= TOL
    assert rel_l2(cpu(snap), f["pdhg_tv_snap40"]) <= TOL
    x = run_pdhg_reference(TomoProblem(proj, f["pdhg_data"]), 120)
    assert rel_l2(cpu(x), f["pdhg_plain_x"]) <= TOL
    with pytest.raises(ValueError):
        run_pdhg_reference(TomoProblem(proj, f["pdhg_data"]), 0)


def _problem_3d(Z=10, size=32, seed=4):
    from paper_2602_09527_b200 import problems
    g = ParallelGeometry.uniform(30, 45)
    proj = Projector(g, size, size, n_slices=Z)
    vol = problems.ellipsoid_phantom(size, 6, seed)[:Z]
    data = cpu(proj.forward(np.ascontiguousarray(vol)))
    data = data + 0.01 * np.random.default_rng(seed).standard_normal(data.shape)
    return TomoProblem(proj, data, tv=TvProxConfig(alpha=0.05, inner_iterations=12)), proj


@pytest.mark.parametrize("slabs,inner", [(2, 12), (3, 12), (5, 12), (10, 12), (2, 13), (3, 14),
                                         (5, 13)])
def test_zslab_decomposition_is_bitwise_identical(slabs, inner):
    """3D z-slab data path emulated on one device: every virtual slab sees its
    neighbours only through the ghost planes the halo exchange fills; the
    trajectory must equal the single-volume run bit for bit (the projector is
    slice-local, the slab FGP recomputes the same values).  Slabs of >= 3
    planes (2, 3 of 10) run the three-iteration column pass with 3-plane
    ghosts exchanged once per pass, the remainder of the iteration count (12,
    13, 14: 0, 1, 2) a single iteration or a two-iteration pass; 2-plane slabs
    (5) the two-iteration pass with 2-plane ghosts; 1-plane slabs (10) the
    one-iteration kernel with a halo round per iteration."""
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200.solvers import _init_state, _plan_segment
    problem, proj = _problem_3d()
    tv = TvProxConfig(alpha=problem.tv.alpha, inner_iterations=inner)
    lip = proj.norm_sq(20, 0)
    outs = []
    for g in (1, slabs):
        cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.5, n_subsets=5, estimator="svrg",
                           max_data_passes=1e9, seed=7)
        st = _init_state(cfg, TomoProblem(proj, problem.data, tv=tv), None)
        if g > 1:
            D.emulate_zslabs(st.session, g)
        subs, th, rf, _, _ = _plan_segment(st, cfg, 1 << 40, max_steps=30)
        assert th.sum() >= 5
        st.session.run(subs, th, rf, 0)
        outs.append((st.x.clone(), st.session.buffer(6).clone()))
    assert torch.equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])


def test_zslab_nccl_on_one_rank_is_bitwise_identical():
    """The z-slab path through a real one-rank NCCL communicator (attach,
    ncclSend/Recv symbols, slab FGP driver with the halo callback)."""
    import socket
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        problem, proj = _problem_3d(Z=6)
        lip = proj.norm_sq(20, 0)
        cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.5, n_subsets=5, estimator="svrg",
                           max_data_passes=9, seed=1)
        a = run(cfg, problem)
        b = run(cfg, TomoProblem(proj, problem.data, tv=problem.tv), data_parallel=True)
        assert torch.equal(a.image, b.image)
        assert a.iterations == b.iterations
    finally:
        dist.destroy_process_group()


_PDL_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r})
from paper_2602_09527_b200 import (ParallelGeometry, Projector, SolverConfig, TomoProblem,
                                   TvProxConfig, default_gamma, problems, run)
g = ParallelGeometry.uniform(120, 181)
proj = Projector(g, 128, 128)
x = problems.ellipse_phantom(128, 6, 1)
b = proj.forward(x).double().cpu().numpy() + 0.01 * np.random.default_rng(1).standard_normal((120, 181))
lip = proj.norm_sq(20, 0)
out = []
for est in ("svrg", "saga", "full"):
    cfg = SolverConfig(gamma=default_gamma(est, lip), skip_probability=0.3,
                       n_subsets=10 if est != "full" else 1, estimator=est,
                       max_data_passes=9, seed=2)
    out.append(run(cfg, TomoProblem(proj, b, tv=TvProxConfig(alpha=0.05, inner_iterations=20))).image.cpu().numpy())
np.save(sys.argv[1], np.stack(out))
"""


def test_programmatic_dependent_launch_is_bitwise_neutral(tmp_path):
    """Overlapping kernel prologues with the predecessor's drain (PDL) must not
    change a single bit of the trajectory (PT_PDL=0 launches serially)."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0", "1"):
        path = tmp_path / f"pdl{flag}_{len(outs)}.npy"
        env = dict(os.environ, PT_PDL=flag)
        subprocess.run([sys.executable, "-c", _PDL_SNIPPET.format(repo=repo), str(path)],
                       check=True, env=env, timeout=300)
        outs.append(np.load(path))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
