"""Multi-process host logic of the angle-sector data parallelism, world size
2 over gloo on CPU (the GPU tier runs on one device; the NCCL data path is
covered on the GPU by the single-device sector emulation in
tests/test_gpu_solver.py)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_09527_b200.geometry import ParallelGeometry, angle_sector, build_staggered_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle as O
        from paper_2602_09527_b200.distributed import share_unique_id
        from paper_2602_09527_b200.solvers import SolverConfig, _plan_segment
        from test_host import _state

        out = {}
        # (1) NCCL unique-id exchange: rank 0's 128 bytes reach every rank
        uid = share_unique_id(lambda: bytes(range(128)), rank)
        out["uid_ok"] = uid == bytes(range(128))

        # (2) every rank draws the identical subset / skip / refresh schedule
        cfg = SolverConfig(gamma=1.0, skip_probability=0.1, n_subsets=10, estimator="svrg",
                           max_data_passes=12, seed=0)
        st = _state(cfg, 180)
        subs, th, rf, passes, _ = _plan_segment(st, cfg, 1)
        sig = torch.tensor([int(subs.sum()), int(th.sum()), int(rf.sum()), len(subs)],
                           dtype=torch.int64)
        lo, hi = sig.clone(), sig.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        out["schedule_ok"] = bool(torch.equal(lo, hi))

        # (3) sector-sharded subset gradient: own angles only, summed = full subset
        O.set_mode("exact")
        g = ParallelGeometry.uniform(36, 47)
        rng = np.random.default_rng(5)
        x = rng.standard_normal((24, 24))
        b = rng.standard_normal((36, 47))
        part = build_staggered_partition(36, 4)
        a_lo, a_hi = angle_sector(36, rank, world)
        worst = 0.0
        for sub in part.subsets:
            own = tuple(a for a in sub if a_lo <= a < a_hi)
            partial = np.zeros((24, 24))
            if own:
                r = O.forward_project(x, g, own) - b[list(own)]
                partial = O.back_project(r, g, (24, 24), own)
            t = torch.tensor(partial)
            dist.all_reduce(t)
            full = O.back_project(O.forward_project(x, g, sub) - b[list(sub)], g, (24, 24), sub)
            worst = max(worst, float(np.abs(t.numpy() - full).max() / np.abs(full).max()))
        out["sector_sum_err"] = worst
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_sector_logic_over_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r]["uid_ok"]
        assert results[r]["schedule_ok"]
        assert results[r]["sector_sum_err"] <= 1e-12


# ---------------------------------------------------------------------------
# z-slab decomposition (3D): the halo protocol of csrc/fgp.cu fgp3d_run,
# restated in float64 numpy per rank with gloo send/recv for the ghost planes,
# must reproduce the single-volume 3D FGP of the oracle.
# ---------------------------------------------------------------------------

def _slab_fgp(v_loc, z0, Zg, lam, inner, nonneg, rank, world):
    import torch
    zl, H, W = v_loc.shape

    def exchange(S, send_lo, send_hi):
        """ghost planes of S ([zl + 2, ...]): plane 0 from rank - 1, plane zl + 1 from rank + 1"""
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send_lo)), rank - 1))
            lo = torch.empty(send_lo.shape, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(send_hi)), rank + 1))
            hi = torch.empty(send_hi.shape, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
        for r in reqs:
            r.wait()
        if rank > 0:
            S[0] = lo.numpy()
        if rank + 1 < world:
            S[zl + 1] = hi.numpy()

    def dt(R, z):  # D^T of R at local plane z (global guards)
        zg = z0 + z
        p, q, w = R[z + 1, 0], R[z + 1, 1], R[z + 1, 2]
        x = np.zeros((H, W))
        x[:-1] -= p[:-1]
        x[1:] += p[:-1]
        x[:, :-1] -= q[:, :-1]
        x[:, 1:] += q[:, :-1]
        if zg < Zg - 1:
            x -= w
        if zg > 0:
            x += R[z, 2]
        return x

    vt = np.zeros((H, W))  # ghost v above
    tmp = np.zeros((zl + 2, H, W))
    tmp[1:zl + 1] = v_loc
    exchange(tmp, v_loc[0], v_loc[-1])
    vt = tmp[zl + 1]
    P = np.zeros((zl + 2, 3, H, W))
    Q = P.copy()
    t, beta_r = 1.0, 0.0
    for k in range(inner):
        R = P + beta_r * (P - Q)
        U = np.zeros((zl + 1, H, W))
        for z in range(zl + 1):
            if z0 + z >= Zg:
                continue
            vz = v_loc[z] if z < zl else vt
            U[z] = vz - lam * dt(R, z)
            if nonneg:
                U[z] = np.maximum(U[z], 0.0)
        Pn = np.zeros_like(P)
        eta = 1.0 / (12.0 * lam)
        for z in range(zl):
            u = U[z]
            gv = np.zeros((H, W)); gv[:-1] = u[1:] - u[:-1]
            gh = np.zeros((H, W)); gh[:, :-1] = u[:, 1:] - u[:, :-1]
            gz = (U[z + 1] - u) if z0 + z < Zg - 1 else np.zeros((H, W))
            ph = R[z + 1, 0] + eta * gv
            qh = R[z + 1, 1] + eta * gh
            wh = R[z + 1, 2] + eta * gz
            nrm = np.maximum(1.0, np.sqrt(ph * ph + qh * qh + wh * wh))
            Pn[z + 1] = np.stack([ph / nrm, qh / nrm, wh / nrm])
        exchange(Pn, Pn[1], Pn[zl])
        tn = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        beta_r = (t - 1.0) / tn
        t = tn
        Q, P = P, Pn
    x = np.stack([v_loc[z] - lam * dt(P, z) for z in range(zl)])
    return np.maximum(x, 0.0) if nonneg else x


def _slab_fgp_passes(v_loc, z0, Zg, lam, inner, nonneg, rank, world, D=2):
    """The native multi-iteration column passes on z-slabs (csrc/fgp.cu,
    fgp3d_ghost_exchange): before each pass of D iterations (D = 3 when every
    slab holds >= 3 planes, else 2) a slab receives the D boundary planes of
    P_k and P_{k-1} of its neighbours (and of v, once per pass depth) into
    D-plane ghost regions, computes P_{k+1} on its planes and D - 1 planes into
    each ghost region, ..., P_{k+D} on its own planes; the remainder of the
    iteration count runs a two-iteration pass and / or one iteration with the
    one-plane protocol.  Restated in float64 numpy over gloo."""
    import torch
    zl, H, W = v_loc.shape
    G = 3  # ghost planes per side; extended plane index e = z + G

    def exchange(A, d):
        """A: [zl + 2G, ...]; the d ghost planes nearest the slab <- the
        neighbours' d boundary planes"""
        reqs, lo, hi = [], None, None
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(A[G:G + d])), rank - 1))
            lo = torch.empty(A[:d].shape, dtype=torch.float64)
            reqs.append(dist.irecv(lo, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(A[G + zl - d:G + zl])),
                                   rank + 1))
            hi = torch.empty(A[:d].shape, dtype=torch.float64)
            reqs.append(dist.irecv(hi, rank + 1))
        for r in reqs:
            r.wait()
        if lo is not None:
            A[G - d:G] = lo.numpy()
        if hi is not None:
            A[G + zl:G + zl + d] = hi.numpy()

    def inside(z):
        return 0 <= z0 + z < Zg

    def u_plane(R, V, z):  # u at local plane z (global guards), extended arrays
        if not inside(z):
            return np.zeros((H, W))
        e, zg = z + G, z0 + z
        p, q, w = R[e, 0], R[e, 1], R[e, 2]
        x = np.zeros((H, W))
        x[:-1] -= p[:-1]
        x[1:] += p[:-1]
        x[:, :-1] -= q[:, :-1]
        x[:, 1:] += q[:, :-1]
        if zg < Zg - 1:
            x -= w
        if zg > 0:
            x += R[e - 1, 2]
        u = V[e] - lam * x
        return np.maximum(u, 0.0) if nonneg else u

    def step(P, Q, beta_r, V, lo, hi):
        """one FGP iteration on local planes [lo, hi): P_{k+1}"""
        R = P + beta_r * (P - Q)
        eta = 1.0 / (12.0 * lam)
        Pn = np.zeros_like(P)
        U = {z: u_plane(R, V, z) for z in range(lo, hi + 1)}
        for z in range(lo, hi):
            if not inside(z):
                continue
            u = U[z]
            gv = np.zeros((H, W)); gv[:-1] = u[1:] - u[:-1]
            gh = np.zeros((H, W)); gh[:, :-1] = u[:, 1:] - u[:, :-1]
            gz = (U[z + 1] - u) if z0 + z < Zg - 1 else np.zeros((H, W))
            e = z + G
            ph = R[e, 0] + eta * gv
            qh = R[e, 1] + eta * gh
            wh = R[e, 2] + eta * gz
            nrm = np.maximum(1.0, np.sqrt(ph * ph + qh * qh + wh * wh))
            Pn[e] = np.stack([ph / nrm, qh / nrm, wh / nrm])
        return Pn

    V = np.zeros((zl + 2 * G, H, W))
    V[G:G + zl] = v_loc
    P = np.zeros((zl + 2 * G, 3, H, W))
    Q = P.copy()
    t, betas = 1.0, []
    for _ in range(inner):
        tn = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
        betas.append((t - 1.0) / tn)
        t = tn
    k, v_depth = 0, 0
    for depth in (D, 2):
        while depth > 1 and k + depth <= inner:
            if v_depth != depth:  # v's ghosts, once per pass depth
                exchange(V, depth)
                v_depth = depth
            exchange(P, depth)
            exchange(Q, depth)
            for i in range(depth):  # iteration k + i on planes [-(depth-1-i), zl + depth-1-i)
                br = 0.0 if k + i == 0 else betas[k + i - 1]
                r = depth - 1 - i
                Q, P = P, step(P, Q, br, V, -r, zl + r)
            k += depth
    if k < inner:
        exchange(P, 1)
        exchange(Q, 1)
        if v_depth == 0:
            exchange(V, 1)
        br = 0.0 if k == 0 else betas[k - 1]
        Q, P = P, step(P, Q, br, V, 0, zl)
    exchange(P, 1)
    R = P
    x = []
    for z in range(zl):
        e, zg = z + G, z0 + z
        p, q, w = R[e, 0], R[e, 1], R[e, 2]
        d = np.zeros((H, W))
        d[:-1] -= p[:-1]
        d[1:] += p[:-1]
        d[:, :-1] -= q[:, :-1]
        d[:, 1:] += q[:, :-1]
        if zg < Zg - 1:
            d -= w
        if zg > 0:
            d += R[e - 1, 2]
        x.append(v_loc[z] - lam * d)
    x = np.stack(x)
    return np.maximum(x, 0.0) if nonneg else x


def _zworker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle as O
        from paper_2602_09527_b200 import Projector, TomoProblem
        from paper_2602_09527_b200.distributed import gather_zslabs, zslab_bounds, zslab_problem
        out = {}
        Z, H, W = 7, 9, 11
        z0, z1 = zslab_bounds(Z, rank, world)
        # (1) slab bounds tile the volume in rank order
        spans = [zslab_bounds(Z, g, world) for g in range(world)]
        out["tiles"] = spans[0][0] == 0 and spans[-1][1] == Z and all(
            spans[g][1] == spans[g + 1][0] for g in range(world - 1))
        # (2) the slab problem: own sinogram rows, own projector depth
        g = ParallelGeometry.uniform(12, 15)
        data = np.arange(12 * Z * 15, dtype=np.float64).reshape(12, Z, 15)
        sp = zslab_problem(TomoProblem(Projector(g, W, H, n_slices=Z), data), z0, z1)
        want = data[:, z0:z1, :]
        if z1 - z0 == 1:
            want = want.reshape(12, 15)
        out["slab_ok"] = (sp.projector.n_slices == z1 - z0 and np.array_equal(sp.data, want))
        # (3) gathered volume
        vol = torch.arange(Z * H * W, dtype=torch.float32).reshape(Z, H, W)
        full = gather_zslabs(vol[z0:z1].clone(), Z)
        out["gather_ok"] = bool(torch.equal(full, vol))
        # (4) the halo protocol of the slab FGP = the single-volume 3D FGP
        rng = np.random.default_rng(2)
        v = rng.standard_normal((Z, H, W))
        for nn in (False, True):
            xs = _slab_fgp(v[z0:z1], z0, Z, 0.3, 12, nn, rank, world)
            xt = gather_zslabs(torch.from_numpy(xs), Z).numpy()
            xo, _ = O.tv_prox(v, 1.0, 0.3, 12, nn)
            out[f"fgp_err_{int(nn)}"] = float(np.abs(xt - xo).max())
        # (5) the two-iteration pass protocol (2-plane ghosts once per pass),
        # even and odd iteration counts
        if min(b - a for a, b in spans) >= 2:
            for inner in (12, 7):
                xs = _slab_fgp_passes(v[z0:z1], z0, Z, 0.3, inner, True, rank, world, 2)
                xt = gather_zslabs(torch.from_numpy(xs), Z).numpy()
                xo, _ = O.tv_prox(v, 1.0, 0.3, inner, True)
                out[f"pass2_err_{inner}"] = float(np.abs(xt - xo).max())
        # (6) the three-iteration pass protocol (3-plane ghosts once per pass,
        # then a two-iteration pass and / or one iteration for the remainder)
        # on a volume whose slabs hold >= 3 planes
        Z3 = 3 * world + 1
        a3, b3 = zslab_bounds(Z3, rank, world)
        v3 = rng.standard_normal((Z3, H, W))
        for inner in (12, 13, 14):
            xs = _slab_fgp_passes(v3[a3:b3], a3, Z3, 0.3, inner, True, rank, world, 3)
            xt = gather_zslabs(torch.from_numpy(xs), Z3).numpy()
            xo, _ = O.tv_prox(v3, 1.0, 0.3, inner, True)
            out[f"pass3_err_{inner}"] = float(np.abs(xt - xo).max())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_zslab_logic_and_halo_protocol_over_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_zworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = results[r]
        assert res["tiles"] and res["slab_ok"] and res["gather_ok"], res
        assert res["fgp_err_0"] <= 1e-12 and res["fgp_err_1"] <= 1e-12, res
        for inner in (12, 7):
            if f"pass2_err_{inner}" in res:
                assert res[f"pass2_err_{inner}"] <= 1e-12, res
        for inner in (12, 13, 14):
            assert res[f"pass3_err_{inner}"] <= 1e-12, res


# ---------------------------------------------------------------------------
# image-row decomposition (2D): host logic and the protocols of the native
# rows mode, restated in numpy over a gloo world
# ---------------------------------------------------------------------------

def _exchange_rows(own, lo_g, hi_g, rank, world):
    """Own rows -> extended array with lo_g / hi_g ghost rows from the ranks
    -+ 1 (the native rows halo: first / last own rows sent, ghosts received)."""
    import torch
    hl, W = own.shape
    ext = np.zeros((lo_g + hl + hi_g, W))
    ext[lo_g:lo_g + hl] = own
    reqs, bufs = [], []
    if rank > 0:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[:lo_g])), rank - 1))
        bufs.append(("lo", torch.empty((lo_g, W), dtype=torch.float64)))
        reqs.append(dist.irecv(bufs[-1][1], rank - 1))
    if rank < world - 1:
        reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(own[hl - hi_g:])), rank + 1))
        bufs.append(("hi", torch.empty((hi_g, W), dtype=torch.float64)))
        reqs.append(dist.irecv(bufs[-1][1], rank + 1))
    for r in reqs:
        r.wait()
    for side, t in bufs:
        if side == "lo":
            ext[:lo_g] = t.numpy()
        else:
            ext[lo_g + hl:] = t.numpy()
    return ext


def _row_fgp(v_own, r0, H, lam, inner, nonneg, rank, world, T=4):
    """Row-slab FGP: T iterations per launch on own rows + T+1 ghost rows a
    side (fewer at the image edge), ghosts refreshed before every launch."""
    G = T + 1
    hl, W = v_own.shape
    lo_g = G if rank > 0 else 0
    hi_g = G if rank < world - 1 else 0
    gi = (r0 - lo_g + np.arange(lo_g + hl + hi_g))[:, None]  # image rows of the extended array
    jj = np.arange(W)[None, :]

    def dt(a, b):
        up = np.zeros_like(a); up[1:] = a[:-1]
        left = np.zeros_like(b); left[:, 1:] = b[:, :-1]
        return (-a * (gi < H - 1) + up * (gi > 0)) - b * (jj < W - 1) + left * (jj > 0)

    def grad(u):
        gv = np.zeros_like(u); gv[:-1] = u[1:] - u[:-1]
        gh = np.zeros_like(u); gh[:, :-1] = u[:, 1:] - u[:, :-1]
        return gv * (gi < H - 1), gh * (jj < W - 1)

    own = slice(lo_g, lo_g + hl)
    v = _exchange_rows(v_own, lo_g, hi_g, rank, world)
    p_own = np.zeros((hl, W)); q_own = np.zeros((hl, W))
    r_own, s_own = p_own, q_own
    eta, t, done = 1.0 / (8.0 * lam), 1.0, 0
    while done < inner:
        p, q, r, s = (_exchange_rows(a, lo_g, hi_g, rank, world)
                      for a in (p_own, q_own, r_own, s_own))
        for _ in range(min(T, inner - done)):
            u = v - lam * dt(r, s)
            if nonneg:
                u = np.maximum(u, 0.0)
            gv, gh = grad(u)
            ph, qh = r + eta * gv, s + eta * gh
            nrm = np.maximum(1.0, np.sqrt(ph * ph + qh * qh))
            pn, qn = ph / nrm, qh / nrm
            tn = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
            beta = (t - 1.0) / tn
            t = tn
            r, s = pn + beta * (pn - p), qn + beta * (qn - q)
            p, q = pn, qn
            done += 1
        p_own, q_own, r_own, s_own = p[own], q[own], r[own], s[own]
    p, q = (_exchange_rows(a, lo_g, hi_g, rank, world) for a in (p_own, q_own))
    x = v - lam * dt(p, q)
    return (np.maximum(x, 0.0) if nonneg else x)[own]


def _rworker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import oracle as O
        from paper_2602_09527_b200 import Projector, TomoProblem, TvProxConfig
        from paper_2602_09527_b200.distributed import (gather_rowslabs, rowslab_bounds,
                                                       rowslab_problem)
        out = {}
        H, W = 29, 17
        r0, r1 = rowslab_bounds(H, rank, world)
        spans = [rowslab_bounds(H, g, world) for g in range(world)]
        out["tiles"] = spans[0][0] == 0 and spans[-1][1] == H and all(
            spans[g][1] == spans[g + 1][0] for g in range(world - 1))
        # the slab problem: a row-slab projector over the whole sinogram
        g = ParallelGeometry.uniform(12, 25)
        data = np.arange(12 * 25, dtype=np.float64).reshape(12, 25)
        sp = rowslab_problem(TomoProblem(Projector(g, W, H), data, tv=TvProxConfig(alpha=0.1)),
                             r0, r1)
        out["slab_ok"] = (sp.projector.shape == (r1 - r0, W)
                          and sp.projector.row_slab == (r0, H) and sp.data is data)
        img = torch.arange(H * W, dtype=torch.float32).reshape(H, W)
        out["gather_ok"] = bool(torch.equal(gather_rowslabs(img[r0:r1].clone(), H), img))
        # forward protocol: own-row partial line integrals summed over ranks
        rng = np.random.default_rng(4)
        x = rng.random((H, W))
        mask = np.zeros((H, W)); mask[r0:r1] = 1.0
        part = torch.from_numpy(O.forward_project(x * mask, g, None))
        dist.all_reduce(part)
        full = O.forward_project(x, g, None)
        out["fwd_err"] = float(np.abs(part.numpy() - full).max() / np.abs(full).max())
        # adjoint protocol: each rank's rows of the whole adjoint of the full residual
        res = rng.standard_normal((12, 25))
        adj = O.back_project(res, g, (H, W), None)
        out["adj_rows"] = adj[r0:r1].shape == (r1 - r0, W)
        # TV prox: the ghost-row protocol = the whole-image FGP
        v = rng.standard_normal((H, W))
        for nn in (False, True):
            xs = _row_fgp(v[r0:r1], r0, H, 0.3, 13, nn, rank, world)
            xt = gather_rowslabs(torch.from_numpy(xs), H).numpy()
            xo, _ = O.tv_prox(v, 1.0, 0.3, 13, nn)
            out[f"fgp_err_{int(nn)}"] = float(np.abs(xt - xo).max())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rows_logic_and_protocols_over_gloo(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        res = results[r]
        assert res["tiles"] and res["slab_ok"] and res["gather_ok"] and res["adj_rows"], res
        assert res["fwd_err"] <= 1e-13, res
        assert res["fgp_err_0"] <= 1e-12 and res["fgp_err_1"] <= 1e-12, res
