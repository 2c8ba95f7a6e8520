"""Multi-GPU data parallelism (one process per GPU): angle sectors or image
rows (2D), z-slabs (slice-stacked 3D).

Image rows (``decomposition="rows"``): rank g owns image rows
[g*H/G, (g+1)*H/G) with a row-slab plan; each forward's partial line
integrals are summed in float64 by ncclAllReduce (8 |S_i| B bytes per step:
0.7 MB at config 2), the gather, ProxSkip step and TV prox touch only the own
rows (ghost rows exchanged with ranks g -+ 1 per FGP launch).  The per-step
exchange is 23x smaller than the sector layout's image-sized allreduce and
the prox is sharded too.

Angle sectors (the 2D default, north_star's layout): rank g of G owns the
contiguous sinogram rows of angles [g*A/G, (g+1)*A/G)
(geometry.angle_sector).  Staggered subsets therefore
split across all ranks, so every stochastic step is parallel; the per-step
partial gradient A_i^T r (4 * n_px bytes) and the snapshot full gradient are
summed by ncclAllReduce inside the native executor on the solver stream; the
image, control variate, SAGA/SVRG state and the TV prox stay replicated and
bitwise identical on every rank (deterministic kernels, identical reduced
bytes).  torch.distributed is only the bootstrap: it ships NCCL's unique id
from rank 0; the library dlopens the same libnccl torch uses.
"""

from __future__ import annotations

import ctypes
import glob
import os

import torch
import torch.distributed as dist

from . import _native as N


def nccl_library_path() -> str:
    """The libnccl.so.2 torch is using (nvidia-nccl wheel), else the system one
    (PT_NCCL_LIB names another build, e.g. the tests' host-staged shim)."""
    if os.environ.get("PT_NCCL_LIB"):
        return os.environ["PT_NCCL_LIB"]
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
        hits = glob.glob(os.path.join(base, "lib", "libnccl.so*"))
        if hits:
            return sorted(hits)[0]
    except Exception:
        pass
    return "libnccl.so.2"


_COMMS: dict = {}  # (process group, rank, world) -> pt_comm handle


def communicator(rank: int | None = None, world: int | None = None, group=None):
    """The library's NCCL communicator for this process group, created once
    per process (rank 0 makes the unique id, torch.distributed ships it) and
    shared by every session; ``release_communicators`` frees them."""
    rank = dist.get_rank(group) if rank is None else rank
    world = dist.get_world_size(group) if world is None else world
    key = (id(group) if group is not None else 0, rank, world)
    handle = _COMMS.get(key)
    if handle is None:
        path = nccl_library_path().encode()

        def make_uid() -> bytes:
            uid = (ctypes.c_uint8 * 128)()
            N.check(N.lib().pt_nccl_unique_id(path, uid), "ncclGetUniqueId")
            return bytes(uid)

        payload = share_unique_id(make_uid, rank, group)
        uid = (ctypes.c_uint8 * 128)(*payload)
        handle = ctypes.c_void_p()
        N.check(N.lib().pt_nccl_comm_create(path, uid, rank, world, ctypes.byref(handle)),
                "nccl_comm_create")
        _COMMS[key] = handle
    return handle


def release_communicators() -> None:
    """Destroy the cached communicators (after the last session using them)."""
    while _COMMS:
        _, handle = _COMMS.popitem()
        N.lib().pt_nccl_comm_destroy(handle)


def attach(session, rank: int | None = None, world: int | None = None,
           group=None) -> None:
    """Attach a native solver session to the process group's NCCL
    communicator (angle sectors: rank g owns angles [gA/G, (g+1)A/G))."""
    N.check(N.lib().pt_session_attach_comm(session.handle, communicator(rank, world, group)),
            "attach")


def share_unique_id(make_uid, rank: int, group=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id, every rank receives it."""
    payload = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(payload, src=0, group=group)
    uid = payload[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def emulate_sectors(session, world: int) -> None:
    """Single-device emulation of `world` angle-sector ranks (test hook)."""
    N.check(N.lib().pt_session_emulate_sectors(session.handle, int(world)), "emulate")


def replicas_identical(x: torch.Tensor, group=None) -> bool:
    """Replica check: every rank's iterate has the same bytes (max == min of a
    bit-pattern checksum over ranks)."""
    v = x.contiguous().view(torch.int32).reshape(-1).to(torch.int64)
    chk = torch.stack([v.sum(), (v * torch.arange(v.numel(), device=v.device) % 1000003).sum()])
    lo, hi = chk.clone(), chk.clone()
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return bool(torch.equal(lo, hi))


# ---------------------------------------------------------------------------
# z-slab decomposition of slice-stacked 3D problems
# ---------------------------------------------------------------------------

def zslab_bounds(n_slices: int, rank: int, world: int) -> tuple[int, int]:
    """Rank g of G owns planes [g Z / G, (g + 1) Z / G) (contiguous, in rank order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if n_slices < world:
        raise ValueError(f"{n_slices} slices cannot be split over {world} ranks")
    return n_slices * rank // world, n_slices * (rank + 1) // world


def zslab_problem(problem, z0: int, z1: int):
    """The slab [z0, z1) of a 3D TomoProblem: same geometry and regulariser,
    its own projector (Z = z1 - z0) and the matching sinogram rows (A, Zl, B)
    (slices never interact in the projector: rotation is about z)."""
    from .projector import Projector
    from .solvers import TomoProblem
    proj = problem.projector
    zl = z1 - z0
    sub = Projector(proj.geometry, proj.width, proj.height, n_slices=zl)
    data = problem.data
    if isinstance(data, torch.Tensor):
        slab = data[:, z0:z1, :].contiguous()
    else:
        import numpy as np
        slab = np.ascontiguousarray(np.asarray(data)[:, z0:z1, :])
    if zl == 1:
        slab = slab.reshape(slab.shape[0], slab.shape[2])
    return TomoProblem(sub, slab, tv=problem.tv, denoiser=problem.denoiser)


def attach_zslab(session, z0: int, z_total: int, rank: int | None = None,
                 world: int | None = None, group=None) -> None:
    """Attach a slab session to the process group's communicator for the z
    halo exchange (ranks hold consecutive slabs in rank order)."""
    N.check(N.lib().pt_session_attach_comm_zslab(session.handle,
                                                 communicator(rank, world, group), int(z0),
                                                 int(z_total)), "attach_zslab")


def emulate_zslabs(session, slabs: int) -> None:
    """Single-device emulation of `slabs` z-slab ranks for the 3D TV prox (test hook)."""
    N.check(N.lib().pt_session_emulate_zslabs(session.handle, int(slabs)), "emulate_zslabs")


def gather_zslabs(x_slab: torch.Tensor, n_slices: int, group=None) -> torch.Tensor:
    """The full (Z, H, W) volume on every rank from each rank's slab (log rows
    and the final image only; padded all_gather over the process group)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H, W = x_slab.shape[-2], x_slab.shape[-1]
    zmax = max(zslab_bounds(n_slices, g, world)[1] - zslab_bounds(n_slices, g, world)[0]
               for g in range(world))
    buf = torch.zeros((zmax, H, W), device=x_slab.device, dtype=x_slab.dtype)
    z0, z1 = zslab_bounds(n_slices, rank, world)
    buf[:z1 - z0] = x_slab.reshape(z1 - z0, H, W)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.empty((n_slices, H, W), device=x_slab.device, dtype=x_slab.dtype)
    for g in range(world):
        a, b = zslab_bounds(n_slices, g, world)
        out[a:b] = parts[g][:b - a]
    return out


# ---------------------------------------------------------------------------
# image-row decomposition of 2D problems
# ---------------------------------------------------------------------------

ROW_GHOST = 9  # ghost rows per side of a slab's TV prox (csrc kRowGhost)


def rowslab_bounds(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Rank g of G owns image rows [g H / G, (g + 1) H / G) (contiguous, rank order)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    if n_rows < world:
        raise ValueError(f"{n_rows} rows cannot be split over {world} ranks")
    return n_rows * rank // world, n_rows * (rank + 1) // world


def rowslab_problem(problem, r0: int, r1: int):
    """Rows [r0, r1) of a 2D TomoProblem: a row-slab projector (partial line
    integrals; the sinogram stays whole), same data and regulariser."""
    from .projector import Projector
    from .solvers import TomoProblem
    proj = problem.projector
    if getattr(proj, "n_slices", 1) != 1:
        raise ValueError("row slabs are a 2D decomposition")
    if problem.tv is not None and r1 - r0 < ROW_GHOST and (r0 > 0 or r1 < proj.height):
        raise ValueError(f"a row slab needs at least {ROW_GHOST} rows for the TV prox")
    sub = Projector(proj.geometry, proj.width, r1 - r0, row_slab=(r0, proj.height))
    return TomoProblem(sub, problem.data, tv=problem.tv, denoiser=problem.denoiser)


def attach_rows(session, r0: int, rows_total: int, rank: int | None = None,
                world: int | None = None, group=None) -> None:
    """Attach a row-slab session to the process group's communicator."""
    N.check(N.lib().pt_session_attach_comm_rows(session.handle,
                                                communicator(rank, world, group), int(r0),
                                                int(rows_total)), "attach_rows")


def gather_rowslabs(x_slab: torch.Tensor, n_rows: int, group=None) -> torch.Tensor:
    """The full (H, W) image on every rank from each rank's rows (log rows and
    the final image only; padded all_gather over the process group)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    W = x_slab.shape[-1]
    spans = [rowslab_bounds(n_rows, g, world) for g in range(world)]
    hmax = max(b - a for a, b in spans)
    buf = torch.zeros((hmax, W), device=x_slab.device, dtype=x_slab.dtype)
    r0, r1 = spans[rank]
    buf[:r1 - r0] = x_slab.reshape(r1 - r0, W)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = torch.empty((n_rows, W), device=x_slab.device, dtype=x_slab.dtype)
    for g, (a, b) in enumerate(spans):
        out[a:b] = parts[g][:b - a]
    return out
