"""The multi-GPU row decomposition of 2D problems, checked on
one device: slab plans (rows [r0, r0 + Hl) of the image) give partial line
integrals that add up to the whole image's, their adjoint is the whole
adjoint's rows, and the row-slab TV prox (ghost rows standing in for the NCCL
halo exchange) equals the whole-image prox bitwise."""

import ctypes

import numpy as np
import pytest
import torch

from conftest import rel_l2
from paper_2602_09527_b200 import ParallelGeometry, Projector, TvProxConfig, tv_prox
from paper_2602_09527_b200 import _native as N

pytestmark = pytest.mark.gpu


def _bounds(H, G):
    return [(H * g // G, H * (g + 1) // G) for g in range(G)]


@pytest.mark.parametrize("H,W,A,B,G", [(64, 48, 30, 80, 3), (257, 300, 45, 400, 4),
                                       (2048, 2048, 60, 2900, 8)])
def test_slab_projector_partials_add_up(H, W, A, B, G):
    g = ParallelGeometry.uniform(A, B)
    rng = np.random.default_rng(H + W)
    x = torch.tensor(rng.random((H, W)), device="cuda", dtype=torch.float32)
    y = torch.tensor(rng.standard_normal((A, B)), device="cuda", dtype=torch.float32)
    full = Projector(g, W, H)
    sub = tuple(range(1, A, 7))
    yf = full.forward(x, sub).double()
    af = full.adjoint(y[list(sub)], sub).double()
    ys = torch.zeros_like(yf)
    nnz = 0
    for r0, r1 in _bounds(H, G):
        p = Projector(g, W, r1 - r0, row_slab=(r0, H))
        ys += p.forward(x[r0:r1].contiguous(), sub).double()
        a = p.adjoint(y[list(sub)], sub).double()
        # float32 positions in different tile frames: the projection tolerance
        assert rel_l2(a.cpu().numpy(), af[r0:r1].cpu().numpy()) <= 1e-5
        nnz += p.plan.nnz(sub)
    assert rel_l2(ys.cpu().numpy(), yf.cpu().numpy()) <= 1e-5
    assert nnz == full.plan.nnz(sub)


@pytest.mark.parametrize("H,W,inner,nn", [(300, 701, 13, True), (2048, 2048, 100, True),
                                          (100, 90, 17, False), (64, 256, 8, True)])
def test_row_slab_tv_prox_is_bitwise_whole_image(H, W, inner, nn):
    rng = np.random.default_rng(H * W)
    v = torch.tensor(rng.standard_normal((H, W)).cumsum(axis=1) * 0.05 + 0.3, device="cuda",
                     dtype=torch.float32)
    lam = 0.05
    x_ref, st = tv_prox(v, 1.0, TvProxConfig(alpha=lam, inner_iterations=inner, nonneg=nn))
    plan = Projector(ParallelGeometry.uniform(4, 8), W, H).plan
    for G in (1, 2, 3, max(1, H // 16)):
        p = torch.zeros_like(v)
        q = torch.zeros_like(v)
        x = torch.empty_like(v)
        N.check(N.lib().pt_tv_prox_emulate_rows(plan.handle, G, N.ptr(v), ctypes.c_double(lam),
                                                inner, int(nn), N.ptr(p), N.ptr(q), N.ptr(x),
                                                N.stream_handle()), "rows prox")
        torch.cuda.synchronize()
        assert torch.equal(x, x_ref), G
        assert torch.equal(p, st.p) and torch.equal(q, st.q), G


def _small_2d(seed=3):
    from paper_2602_09527_b200 import problems
    g = ParallelGeometry.uniform(36, 60)
    proj = Projector(g, 40, 48)
    img = problems.ellipse_phantom(48, 6, seed)[:, 4:44]
    data = proj.forward(np.ascontiguousarray(img)).double().cpu().numpy()
    data = data + 0.01 * np.random.default_rng(seed).standard_normal(data.shape)
    return proj, data


@pytest.mark.parametrize("estimator", ["svrg", "saga"])
def test_rows_nccl_on_one_rank_is_bitwise_identical(estimator):
    """The image-rows data path through a real one-rank NCCL communicator
    (row-slab plan covering the image, float64 partial line integrals ->
    ncclAllReduce -> residual finish kernel -> own-row gather, the row-slab TV
    prox with its halo callback): bitwise the single-GPU trajectory."""
    import socket
    import torch.distributed as dist
    from paper_2602_09527_b200 import SolverConfig, TomoProblem, run
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        proj, data = _small_2d()
        lip = proj.norm_sq(20, 0)
        tv = TvProxConfig(alpha=0.02, inner_iterations=20)
        cfg = SolverConfig(gamma=1.0 / lip if estimator == "svrg" else 1.0 / (3 * lip),
                           skip_probability=0.3, n_subsets=6, estimator=estimator,
                           max_data_passes=12, seed=5)
        a = run(cfg, TomoProblem(proj, data, tv=tv))
        b = run(cfg, TomoProblem(proj, data, tv=tv), data_parallel=True, decomposition="rows")
        assert torch.equal(a.image, b.image)
        assert a.iterations == b.iterations
        assert b.rows[-1][5] > 0  # prox calls happened
    finally:
        dist.destroy_process_group()


def test_rows_snapshot_residual_on_a_nonzero_rank():
    """In the rows layout every rank owns every angle, so the SVRG snapshot
    residual A x_snap - b is indexed from angle 0 on every rank (it was once
    offset by the angle-sector start A*rank/world).  A one-rank communicator
    whose session is told it is rank 1 of 2 (no TV prox, so no halo traffic)
    must reproduce the single-GPU SVRG trajectory bit for bit."""
    import socket
    import torch.distributed as dist
    from paper_2602_09527_b200 import SolverConfig, TomoProblem
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200.solvers import _init_state, _plan_segment
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        proj, data = _small_2d()
        lip = proj.norm_sq(20, 0)
        cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.3, n_subsets=6, estimator="svrg",
                           max_data_passes=1e9, seed=5)
        outs = []
        for rows in (False, True):
            problem = TomoProblem(proj, data)
            if rows:
                H = proj.height
                st = _init_state(cfg, D.rowslab_problem(problem, 0, H), None,
                                 rowslab=(0, H, H))
                N.check(N.lib().pt_session_override_rank(st.session.handle, 1, 2), "override")
                st.session.init()
            else:
                st = _init_state(cfg, problem, None)
            subs, th, rf, _, _ = _plan_segment(st, cfg, 1 << 40, max_steps=20)
            assert rf.any()  # a refresh inside the segment
            st.session.run(subs, th, rf, 0)
            outs.append(st.x.clone())
        assert torch.equal(outs[0], outs[1])
    finally:
        dist.destroy_process_group()
