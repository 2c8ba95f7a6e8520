"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (the reference is importable read-only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--c1]

Every fixture is produced by the reference package ``proxtomo``
(arxiv/paper_2602_09527) through its public API; the only non-reference
input is the BASELINE phantom law of paper_2602_09527_b200/problems.py
(numpy-only, deterministic), because the reference has no generator for it.
The GPU box never runs this script (no /root/reference there); tests load
the .npz files it wrote.
"""

from __future__ import annotations

import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import proxtomo as P  # noqa: E402  (the reference)
from proxtomo.regularizers import TvProxConfig, tv_prox  # noqa: E402
from proxtomo.solvers import (SolverConfig, TomoProblem, _init_state,  # noqa: E402
                              default_gamma, run)

from paper_2602_09527_b200 import problems  # noqa: E402  (host-only phantom law)

PROJ_CASES = [
    # (H, W, A, B, bin_spacing, pixel_size, subset)
    (64, 64, 60, 95, 1.0, 1.0, (1, 7, 13, 30, 44, 59)),
    (40, 48, 36, 71, 1.0, 1.0, tuple(range(0, 36, 5))),
    (33, 33, 180, 47, 1.0, 1.0, tuple(range(3, 180, 10))),
    (16, 16, 10, 23, 1.0, 1.0, (0, 5)),
    (20, 24, 13, 31, 0.7, 1.3, (2, 3, 11)),
    (31, 17, 45, 40, 1.5, 1.0, tuple(range(0, 45, 4))),
    (1, 1, 1, 1, 1.0, 2.0, (0,)),
    (128, 128, 180, 192, 1.0, 1.0, tuple(range(0, 180, 10))),
]


def projector_fixtures():
    rng = np.random.default_rng(20260101)
    out = {}
    for ci, (H, W, A, B, ds, h, sub) in enumerate(PROJ_CASES):
        g = P.ParallelGeometry.uniform(A, B, ds, h)
        x = rng.standard_normal((H, W))
        y = rng.standard_normal((A, B))
        ys = rng.standard_normal((len(sub), B))
        out[f"p{ci}_meta"] = np.array([H, W, A, B, ds, h], dtype=np.float64)
        out[f"p{ci}_subset"] = np.array(sub, dtype=np.int64)
        out[f"p{ci}_x"] = x
        out[f"p{ci}_ys"] = ys
        if H * W <= 4096:  # full-operator goldens only for the small grids (size cap)
            out[f"p{ci}_y"] = y
            out[f"p{ci}_fwd"] = P.forward_project(x, g)
            out[f"p{ci}_adj"] = P.back_project(y, g, (H, W))
        out[f"p{ci}_fwd_sub"] = P.forward_project(x, g, sub)
        out[f"p{ci}_adj_sub"] = P.back_project(ys, g, (H, W), sub)
        out[f"p{ci}_nnz_sub"] = np.array(P.projector._tables(g, W, H).pair(sub)[0].nnz)
    # operator norms (projector.py:183-197)
    for key, (A, B, W, H, it, seed) in {"norm_desk": (60, 95, 64, 64, 50, 0),
                                         "norm_small": (10, 23, 16, 16, 100, 0)}.items():
        out[key] = np.array(P.operator_norm_sq(P.ParallelGeometry.uniform(A, B), W, H, it, seed))
    return out


def fgp_fixtures():
    rng = np.random.default_rng(7)
    out = {}
    u = rng.standard_normal((17, 23))
    out["fgp_u"] = u
    for nn in (0, 1):
        cfg = TvProxConfig(alpha=0.5, inner_iterations=37, nonneg=bool(nn))
        x, st = tv_prox(u, 0.8, cfg)
        xw, stw = tv_prox(u, 0.8, cfg, warm=st)
        out[f"fgp_x_nn{nn}"] = x
        out[f"fgp_p_nn{nn}"] = st.p
        out[f"fgp_q_nn{nn}"] = st.q
        out[f"fgp_xw_nn{nn}"] = xw
    # config-size case where the prox moves the image by O(1e-1)
    img = problems.ellipse_phantom(128, 10, 3) + 0.05 * rng.standard_normal((128, 128))
    out["fgp128_v"] = img
    cfg = TvProxConfig(alpha=0.02, inner_iterations=50)
    x, st = tv_prox(img, 1.0, cfg)
    out["fgp128_x"] = x
    x2, _ = tv_prox(img, 1.0, cfg, warm=st)
    out["fgp128_x_warm"] = x2
    return out


def schedule_fixtures():
    """The reference's own subset / skip draws (solvers.py:164,174-176,198-238)."""
    out = {}
    for name, (n, p, k, seed) in {"c0": (10, 0.1, 500, 0), "c1": (20, 0.05, 2000, 0),
                                  "c2": (60, 0.05, 1800, 0), "c3": (40, 0.1, 800, 0),
                                  "s23": (5, 0.4, 300, 23)}.items():
        ss = np.random.SeedSequence(seed).spawn(3)
        rs, rt = np.random.default_rng(ss[0]), np.random.default_rng(ss[1])
        subs = np.array([int(rs.integers(n)) for _ in range(k)])
        th = np.array([bool(rt.random() < p) for _ in range(k)])
        out[f"sched_{name}_subsets"] = subs
        out[f"sched_{name}_theta"] = th
    # loopless refresh stream (estimators.py:158-162)
    ss = np.random.SeedSequence(4).spawn(3)
    rr = np.random.default_rng(ss[2])
    out["sched_lsvrg_refresh"] = np.array([bool(rr.random() < 0.2) for _ in range(400)])
    return out


def small_run_fixtures():
    """Whole reference runs on the 16x16 small problem (tests/conftest.py:50-63)."""
    g = P.ParallelGeometry.uniform(10, 23)
    proj = P.Projector(g, 16, 16)
    rng = np.random.default_rng(0)
    truth = np.zeros((16, 16))
    truth[4:12, 5:11] = 1.0
    data = proj.forward(truth) + 0.1 * rng.standard_normal((10, 23))
    tv = TvProxConfig(alpha=0.5, inner_iterations=10)
    problem = TomoProblem(proj, data, tv=tv)
    lip = proj.norm_sq(iterations=100, seed=0)
    out = {"small_data": data, "small_L": np.array(lip)}
    for est, p, passes, seed in (("full", 1.0, 20, 1), ("sgd", 0.4, 30, 17), ("saga", 0.4, 30, 3),
                                 ("svrg", 0.4, 30, 23), ("lsvrg", 0.5, 30, 4), ("svrg", 1.0, 15, 5)):
        gamma = default_gamma(est, lip)
        cfg = SolverConfig(gamma=gamma, skip_probability=p, n_subsets=5 if est != "full" else 1,
                           estimator=est, max_data_passes=passes, seed=seed)
        rec = run(cfg, problem, record_objective=True)
        tag = f"small_{est}_p{p}_s{seed}"
        out[tag + "_image"] = rec.image
        out[tag + "_passes"] = rec.column("data_passes")
        out[tag + "_prox"] = rec.column("prox_calls")
        out[tag + "_obj"] = rec.column("objective")
        out[tag + "_iters"] = np.array(rec.iterations)
    return out


def pdhg_fixtures():
    """The reference's PDHG solver (solvers.py:395-455) on the small problem,
    with and without TV; a snapshot part-way."""
    from proxtomo.solvers import run_pdhg_reference
    g = P.ParallelGeometry.uniform(10, 23)
    proj = P.Projector(g, 16, 16)
    rng = np.random.default_rng(0)
    truth = np.zeros((16, 16))
    truth[4:12, 5:11] = 1.0
    data = proj.forward(truth) + 0.1 * rng.standard_normal((10, 23))
    out = {"pdhg_data": data}
    x, snap = run_pdhg_reference(TomoProblem(proj, data, tv=TvProxConfig(alpha=0.5)), 300,
                                 snapshot_at=40)
    out["pdhg_tv_x"], out["pdhg_tv_snap40"] = x, snap
    out["pdhg_plain_x"] = run_pdhg_reference(TomoProblem(proj, data), 120)
    return out


def fista_fixtures():
    """The reference's run_fista / run_ista (solvers.py:339-392): the 16x16
    small problem (TV, 40 passes; and without a regulariser) and 20 FISTA
    passes of BASELINE config 0 from its golden problem."""
    from proxtomo.solvers import run_fista, run_ista
    g = P.ParallelGeometry.uniform(10, 23)
    proj = P.Projector(g, 16, 16)
    rng = np.random.default_rng(0)
    truth = np.zeros((16, 16))
    truth[4:12, 5:11] = 1.0
    data = proj.forward(truth) + 0.1 * rng.standard_normal((10, 23))
    lip = proj.norm_sq(iterations=100, seed=0)
    out = {}
    for tag, tv in (("tv", TvProxConfig(alpha=0.5, inner_iterations=10)), ("plain", None)):
        problem = TomoProblem(proj, data, tv=tv)
        for name, fn in (("fista", run_fista), ("ista", run_ista)):
            rec = fn(SolverConfig(gamma=1.0 / lip, max_data_passes=40, seed=0), problem,
                     record_objective=True)
            key = f"small_{name}_{tag}"
            out[key + "_image"] = rec.image
            out[key + "_obj"] = rec.column("objective")
            out[key + "_prox"] = rec.column("prox_calls")
            out[key + "_iters"] = np.array(rec.iterations)
    c0 = np.load(os.path.join(HERE, "reference_c0.npz"))
    cfg = problems.CONFIGS["c0"]
    proj = P.Projector(P.ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins), cfg.size, cfg.size)
    problem = TomoProblem(proj, c0["c0_b"], tv=TvProxConfig(alpha=float(c0["c0_alpha"]),
                                                            inner_iterations=cfg.fgp_inner))
    rec = run_fista(SolverConfig(gamma=1.0 / float(c0["c0_L"]), max_data_passes=20, seed=0),
                    problem, record_objective=True)
    out["c0_fista_image"] = rec.image
    out["c0_fista_obj"] = rec.column("objective")
    out["c0_fista_iters"] = np.array(rec.iterations)
    return out


def config_run(name: str, record_objective=True):
    cfg = problems.CONFIGS[name]
    g = P.ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = P.Projector(g, cfg.size, cfg.size)
    x_true = problems.phantom_for(cfg)
    clean = proj.forward(x_true)
    b = problems.add_noise(clean, cfg.noise, cfg.noise_seed)
    atb = proj.adjoint(b)
    alpha = problems.alpha_from_backprojection(float(np.abs(atb).max()), cfg.n_pixels)
    lip = proj.norm_sq(iterations=cfg.power_iterations, seed=cfg.power_seed)
    gamma = default_gamma(cfg.estimator, lip)
    tv = TvProxConfig(alpha=alpha, inner_iterations=cfg.fgp_inner)
    problem = TomoProblem(proj, b, tv=tv)
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=cfg.max_data_passes,
                        seed=cfg.solver_seed)
    # pre-warm the CSR tables and every subset pair
    tables = P.projector._tables(g, cfg.size, cfg.size)
    for sub in P.build_staggered_partition(cfg.n_angles, cfg.n_subsets).subsets:
        tables.pair(sub)
    t0 = time.perf_counter()
    rec = run(scfg, problem, record_objective=record_objective)
    wall = time.perf_counter() - t0
    out = {f"{name}_b": b, f"{name}_L": np.array(lip), f"{name}_alpha": np.array(alpha),
           f"{name}_gamma": np.array(gamma), f"{name}_image": rec.image,
           f"{name}_passes": rec.column("data_passes"), f"{name}_prox": rec.column("prox_calls"),
           f"{name}_iters": np.array(rec.iterations),
           f"{name}_work_seconds": np.array(rec.rows[-1][1]), f"{name}_wall": np.array(wall)}
    if record_objective:
        out[f"{name}_obj"] = rec.column("objective")
    return out


def main():
    fx = {}
    fx.update(projector_fixtures())
    fx.update(fgp_fixtures())
    fx.update(schedule_fixtures())
    np.savez_compressed(os.path.join(HERE, "reference_units.npz"), **fx)
    np.savez_compressed(os.path.join(HERE, "reference_small_runs.npz"), **small_run_fixtures())
    np.savez_compressed(os.path.join(HERE, "reference_pdhg.npz"), **pdhg_fixtures())
    if "--pdhg-only" in sys.argv:
        return
    if "--fista-only" in sys.argv:
        np.savez_compressed(os.path.join(HERE, "reference_fista.npz"), **fista_fixtures())
        return
    if "--c1-only" not in sys.argv:
        c0 = config_run("c0")
        np.savez_compressed(os.path.join(HERE, "reference_c0.npz"), **c0)
        np.savez_compressed(os.path.join(HERE, "reference_fista.npz"), **fista_fixtures())
        print("c0 reference work_seconds", float(c0["c0_work_seconds"]), "prox",
              c0["c0_prox"][-1], "iters", c0["c0_iters"][-1])
    if "--c1" in sys.argv or "--c1-only" in sys.argv:
        # config 1 (512^2 SAGA, 100 epochs): minutes and ~18 GiB; store the
        # final image as float32 plus the row columns
        c1 = config_run("c1", record_objective=True)  # objective at each of the 101 rows
        c1["c1_image"] = c1["c1_image"].astype(np.float32)
        # b is not stored (size cap): tests regenerate it with the pinned oracle
        # forward (<= 1e-14 of the reference's) and the same noise draw
        del c1["c1_b"]
        np.savez_compressed(os.path.join(HERE, "reference_c1.npz"), **c1)
        print("c1 reference work_seconds", float(c1["c1_work_seconds"]))


if __name__ == "__main__":
    main()
