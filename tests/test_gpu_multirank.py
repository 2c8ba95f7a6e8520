"""The library's real multi-rank data paths with 2-3 ranks on ONE GPU.

The ranks are processes sharing cuda:0; their communicator is
``tests/nccl_shim.c`` loaded in place of libnccl.so.2 (PT_NCCL_LIB): every
ncclAllReduce / ncclSend / ncclRecv synchronises the caller's stream and
exchanges host copies through files, so ranks wait for each other on the host
and never inside a kernel.  What runs is the product's own multi-rank code:
communicator creation from a unique id shipped over torch.distributed (gloo),
the sharded selections, the per-step partial-gradient allreduce (angle
sectors), the float64 line-integral allreduce and the ghost-row exchange
(image rows), the 2-plane ghost exchange of the 3D column pass (z-slabs), and
the rank-side gathers of the final image.  The shim sums in rank order, as the
single-device sector emulation does, so sector runs are compared bit for bit.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    out = tmp_path_factory.mktemp("shim")
    so = out / "libnccl_shim.so"
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-O2", "-shared", "-fPIC", f"-I{cuda}/include",
                    os.path.join(REPO, "tests", "nccl_shim.c"), "-o", str(so),
                    f"-L{cuda}/lib64/stubs", "-lcuda"], check=True)
    return str(so)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


_COMMON = r"""
import os, sys, numpy as np, torch
sys.path.insert(0, {repo!r})
import torch.distributed as dist
from paper_2602_09527_b200 import (ParallelGeometry, Projector, SolverConfig, TomoProblem,
                                   TvProxConfig, default_gamma, problems, run)
from paper_2602_09527_b200 import distributed as D
from paper_2602_09527_b200.solvers import _full_gradient_config, _init_state, _plan_segment
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
out = sys.argv[1]


def problem_2d():
    g = ParallelGeometry.uniform(120, 97)
    proj = Projector(g, 64, 64)
    x_true = problems.ellipse_phantom(64, 6, 2)
    data = proj.forward(x_true).cpu().numpy() + 0.01 * np.random.default_rng(0).standard_normal((120, 97))
    return proj, data, TvProxConfig(alpha=0.2, inner_iterations=10)


def problem_3d():
    g = ParallelGeometry.uniform(30, 45)
    proj = Projector(g, 32, 32, n_slices=10)
    vol = np.ascontiguousarray(problems.ellipsoid_phantom(32, 6, 4)[:10])
    data = proj.forward(vol).cpu().numpy()
    data = data + 0.01 * np.random.default_rng(4).standard_normal(data.shape)
    return proj, data, TvProxConfig(alpha=0.05, inner_iterations=12)


def sector_steps(est, emulate):
    # the sector data path: K steps of one planned segment (draws fixed by the seed)
    proj, data, tv = problem_2d()
    lip = proj.norm_sq(30, 0)
    kind = None
    if est == "fista":
        kind = "fista"
        cfg = _full_gradient_config(SolverConfig(gamma=1.0 / lip, max_data_passes=1e9))
    else:
        cfg = SolverConfig(gamma=default_gamma(est, lip), skip_probability=0.3,
                           n_subsets=6 if est != "full" else 1, estimator=est,
                           max_data_passes=1e9, seed=3)
    st = _init_state(cfg, TomoProblem(proj, data, tv=tv), None, data_parallel=not emulate,
                     kind=kind)
    if emulate:
        D.emulate_sectors(st.session, world)
        if est in ("svrg", "lsvrg"):
            st.session.init()  # snapshot gradient through the sectors
    subs, th, rf, _, _ = _plan_segment(st, cfg, 1 << 40, max_steps=40)
    assert th.sum() >= 5 or kind == "fista"
    st.session.run(subs, th, rf, 0)
    return st.x.cpu().numpy()
"""

_RANK = _COMMON + r"""
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + os.environ["PORT"],
                        rank=rank, world_size=world)
torch.cuda.set_device(0)
kind, arg = sys.argv[2], sys.argv[3]
if kind == "sectors":
    np.save(out, sector_steps(arg, emulate=False))
else:
    if kind == "zslab":
        proj, data, tv = problem_3d()
    else:
        proj, data, tv = problem_2d()
    lip = proj.norm_sq(30, 0)
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.5, n_subsets=5, estimator=arg,
                       max_data_passes=9, seed=1)
    rec = run(cfg, TomoProblem(proj, data, tv=tv), data_parallel=True,
              decomposition="rows" if kind == "rows" else "sectors")
    np.savez(out, image=rec.image.cpu().numpy(), iters=np.array(rec.iterations),
             prox=rec.column("prox_calls"))
D.release_communicators()
dist.destroy_process_group()
"""

_SINGLE = _COMMON + r"""
kind, arg = sys.argv[2], sys.argv[3]
if kind == "sectors":
    np.save(out, sector_steps(arg, emulate=True))
else:
    proj, data, tv = problem_3d() if kind == "zslab" else problem_2d()
    lip = proj.norm_sq(30, 0)
    cfg = SolverConfig(gamma=1.0 / lip, skip_probability=0.5, n_subsets=5, estimator=arg,
                       max_data_passes=9, seed=1)
    rec = run(cfg, TomoProblem(proj, data, tv=tv))
    np.savez(out, image=rec.image.cpu().numpy(), iters=np.array(rec.iterations),
             prox=rec.column("prox_calls"))
"""


def _launch(shim, tmp_path, world, kind, arg, extra_env=None):
    """Run `world` rank processes on cuda:0 and the single-device reference;
    returns (per-rank outputs, reference output) paths."""
    port = _free_port()
    shim_dir = tmp_path / "rdv"
    shim_dir.mkdir(exist_ok=True)
    ext = ".npy" if kind == "sectors" else ".npz"
    procs, outs = [], []
    for r in range(world):
        path = str(tmp_path / f"{kind}_{arg}_w{world}_r{r}{ext}")
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), PORT=str(port),
                   MASTER_ADDR="127.0.0.1", PT_NCCL_LIB=shim, PT_NCCL_SHIM_DIR=str(shim_dir),
                   **(extra_env or {}))
        procs.append(subprocess.Popen([sys.executable, "-c", _RANK.format(repo=REPO), path,
                                       kind, arg], env=env))
        outs.append(path)
    try:
        for p in procs:
            assert p.wait(timeout=600) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    # the ranks' communicator was the shim (its rendezvous directory exists)
    assert any(d.name.startswith("shim_") for d in shim_dir.iterdir())
    ref = str(tmp_path / f"{kind}_{arg}_w{world}_single{ext}")
    env = dict(os.environ, RANK="0", WORLD_SIZE=str(world))
    subprocess.run([sys.executable, "-c", _SINGLE.format(repo=REPO), ref, kind, arg], env=env,
                   check=True, timeout=600)
    return outs, ref


@pytest.mark.parametrize("est,world,prox", [("svrg", 2, "1"), ("saga", 3, "1"), ("full", 2, "1"),
                                            ("fista", 3, "1"), ("svrg", 3, "0")])
def test_angle_sectors_multirank_match_emulation_bitwise(shim, tmp_path, est, world, prox):
    """Real sector ranks (own angles, partial A_i^T r, rank-order allreduce,
    shared epilogue; the TV prox sharded by image rows with ghost-row
    exchanges and the new rows broadcast to every rank, or replicated with
    PT_SECTOR_PROX=0): every rank's iterate equals the single-device emulation
    of the same sectors bit for bit."""
    outs, ref = _launch(shim, tmp_path, world, "sectors", est, {"PT_SECTOR_PROX": prox})
    # the sharded prox ran exactly when enabled (its row broadcasts)
    assert bool(list((tmp_path / "rdv").glob("shim_*/bc_*"))) == (prox == "1")
    want = np.load(ref)
    for path in outs:
        assert np.array_equal(np.load(path), want)


def test_zslab_multirank_matches_single_volume_bitwise(shim, tmp_path):
    """3D z-slabs on 2 real ranks (5 planes each: the two-iteration column pass
    with 2-plane ghosts sent / received once per pass, slab snapshots, gathered
    volume): run() equals the single-volume run bit for bit."""
    outs, ref = _launch(shim, tmp_path, 2, "zslab", "svrg")
    want = np.load(ref)
    for path in outs:
        got = np.load(path)
        assert np.array_equal(got["image"], want["image"])
        assert np.array_equal(got["iters"], want["iters"])
        assert np.array_equal(got["prox"], want["prox"])


@pytest.mark.parametrize("est", ["svrg", "saga"])
def test_image_rows_multirank_match_single_device(shim, tmp_path, est):
    """2D image rows on 2 real ranks (row-slab plans, float64 line-integral
    allreduce, ghost-row exchange per FGP launch, gathered image): the
    single-device trajectory up to the order of the float64 line-integral sums."""
    outs, ref = _launch(shim, tmp_path, 2, "rows", est)
    want = np.load(ref)
    for path in outs:
        got = np.load(path)
        err = np.linalg.norm(got["image"] - want["image"]) / np.linalg.norm(want["image"])
        assert err <= 1e-5
        assert np.array_equal(got["iters"], want["iters"])
        assert np.array_equal(got["prox"], want["prox"])
