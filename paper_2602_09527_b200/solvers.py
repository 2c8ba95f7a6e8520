"""ProxSkip driver with variance-reduced estimators, executed natively.

Drop-in for pkg/src/proxtomo/solvers.py (``SolverConfig``, ``TomoProblem``,
``IterateState``, ``RunRecord``, ``DivergenceError``, ``proxskip_step``,
``run``, ``run_ista``, ``run_fista``, ``composite_objective``,
``default_gamma``, ``fista_gamma``, ``optimal_p``).

Division of labour:
  * host (this file): the reference's control flow, bit-exact -- the three
    PCG64 streams from SeedSequence(seed).spawn(3) (:164,174-176), the subset /
    skip / refresh draws (:198-214,238; estimators.py:149-162), float64 data
    pass accounting and the log-row schedule (:302-322);
  * device (csrc/session.cu): the whole iteration -- forward, fused
    gather + estimator + ProxSkip step, FGP prox with the h update -- for a
    whole segment of iterations between two log rows, with no host sync.
Timing: ``wall_seconds`` is device time of the step segments measured with
CUDA events on the solver stream; metric evaluation at rows is excluded, as
the reference's perf_counter brackets only the steps (:304-313).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import estimators as est
from .geometry import SubsetPartition, build_staggered_partition
from .metrics import psnr as _psnr
from .metrics import relative_error_sq as _relative_error_sq
from .metrics import ssim as _ssim
from .projector import Projector, as_device
from .regularizers import TvDualState, TvProxConfig, tv_value

RUN_COLUMNS = ("data_passes", "wall_seconds", "rel_err", "psnr", "ssim",
               "prox_calls", "objective")
INT64_MAX = 2**63 - 1


class DivergenceError(RuntimeError):
    """Iterate became non-finite; carries the partial run record (:42-51)."""

    def __init__(self, iteration: int, gamma: float, record=None):
        super().__init__(f"non-finite iterate at iteration {iteration} (gamma={gamma:g})")
        self.iteration = iteration
        self.gamma = gamma
        self.record = record


@dataclass(frozen=True)
class SolverConfig:
    """One solver run: step size, skipping probability, estimator, budgets (:54-80)."""

    gamma: float
    skip_probability: float = 1.0
    n_subsets: int = 1
    estimator: str = "full"
    max_data_passes: float = 200.0
    tolerance: float | None = None
    time_budget: float | None = None
    mu: float | None = None
    seed: int = 0

    def __post_init__(self):
        if self.gamma <= 0.0:
            raise ValueError("gamma must be positive")
        if not 0.0 < self.skip_probability <= 1.0:
            raise ValueError("skip_probability must be in (0, 1]")
        if self.estimator not in est.ESTIMATOR_KINDS:
            raise ValueError(f"unknown estimator {self.estimator!r}")
        if self.n_subsets < 1:
            raise ValueError("n_subsets must be >= 1")
        if self.max_data_passes <= 0.0:
            raise ValueError("max_data_passes must be positive")
        if self.time_budget is not None and self.time_budget <= 0.0:
            raise ValueError("time_budget must be positive")


@dataclass
class TomoProblem:
    """Measured sinogram, its projector and the regulariser (:83-105).

    ``data`` may be a host array or a CUDA tensor; it is moved to the device
    (float32) on first use by a solver, so a host sinogram's H2D copy is part
    of the solve.  Plug-and-play ``denoiser`` problems are out of scope."""

    projector: Projector
    data: object
    tv: TvProxConfig | None = None
    denoiser: object | None = None

    def __post_init__(self):
        geometry = self.projector.geometry
        shape = tuple(self.data.shape)
        nz = getattr(self.projector, "n_slices", 1)
        want = ((geometry.n_angles, geometry.n_bins) if nz == 1
                else (geometry.n_angles, nz, geometry.n_bins))
        if shape != want:
            raise ValueError(f"data shape {shape} does not match geometry {want}")
        if self.tv is not None and self.denoiser is not None:
            raise ValueError("choose either tv or denoiser, not both")
        self._device_data = None

    def device_data(self) -> torch.Tensor:
        if self._device_data is None:
            if isinstance(self.data, torch.Tensor):
                self._device_data = self.data.to(device="cuda", dtype=torch.float32,
                                                 non_blocking=True).contiguous()
            else:
                self._device_data = as_device(self.data)
        return self._device_data


class _Session:
    """Owner of a native pt_session (device-resident solver state)."""

    def __init__(self, config: SolverConfig, problem: TomoProblem, x0, stream,
                 kind: str | None = None):
        if problem.denoiser is not None:
            raise NotImplementedError("plug-and-play denoisers are out of scope (DESIGN.md)")
        lib = N.lib()
        self.plan = problem.projector.plan
        self.data = problem.device_data()
        self.stream = stream
        tv = problem.tv
        # kind: the session's step ("fista" for run_fista; default the estimator)
        code = N.SESSION_KINDS[kind] if kind else N.EST_CODES[config.estimator]
        desc = N.SolverDesc(code, int(config.n_subsets),
                            float(config.gamma), float(config.skip_probability),
                            1 if tv is not None else 0, float(tv.alpha) if tv else 0.0,
                            int(tv.inner_iterations) if tv else 0,
                            int(bool(tv.warm_start)) if tv else 0,
                            int(bool(tv.nonneg)) if tv else 0)
        self.x0 = None if x0 is None else as_device(x0)
        # every session buffer comes from torch's caching allocator (on the solver
        # stream), so repeated solves reuse memory instead of cudaMalloc-ing ~1 GB
        nbytes = int(lib.pt_session_workspace_bytes(self.plan.handle, ctypes.byref(desc)))
        if nbytes <= 0:
            N.check(N.PT_EINVAL, "session workspace size")
        with torch.cuda.stream(stream):
            self._memory = torch.empty(nbytes + 256, dtype=torch.uint8, device="cuda")
        base = (self._memory.data_ptr() + 255) & ~255
        handle = ctypes.c_void_p()
        N.check(lib.pt_session_create_in(self.plan.handle, ctypes.byref(desc), N.ptr(self.data),
                                         N.ptr(self.x0), base, nbytes, ctypes.byref(handle),
                                         N.stream_handle(stream)), "session")
        self.handle = handle
        self.shape = problem.projector.shape
        self.n = int(np.prod(self.shape))

    def __del__(self):
        try:
            if getattr(self, "handle", None) and N._lib is not None:
                N._lib.pt_session_destroy(self.handle)
        except Exception:
            pass

    def init(self):
        N.check(N.lib().pt_session_init(self.handle, N.stream_handle(self.stream)), "init")

    def run(self, subs: np.ndarray, thetas: np.ndarray, refresh: np.ndarray, k0: int):
        n = len(subs)
        if n == 0:
            return
        s = np.ascontiguousarray(subs, dtype=np.int32)
        t = np.ascontiguousarray(thetas, dtype=np.uint8)
        r = np.ascontiguousarray(refresh, dtype=np.uint8)
        N.check(N.lib().pt_session_run(
            self.handle, n, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), int(k0),
            N.stream_handle(self.stream)), "run")

    def run_marked(self, subs, thetas, refresh, k0: int, marks, events):
        """Enqueue all steps in one native call; events[m] is recorded on the
        session stream after step marks[m] (cumulative step counts)."""
        n = len(subs)
        s = np.ascontiguousarray(subs, dtype=np.int32)
        t = np.ascontiguousarray(thetas, dtype=np.uint8)
        r = np.ascontiguousarray(refresh, dtype=np.uint8)
        mk = np.ascontiguousarray(marks, dtype=np.int32)
        ev = (ctypes.c_void_p * len(events))(*[int(e.cuda_event) for e in events])
        N.check(N.lib().pt_session_run_marked(
            self.handle, n, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
            t.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
            r.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), int(k0), len(mk),
            mk.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ev,
            N.stream_handle(self.stream)), "run")

    def view(self, address) -> torch.Tensor:
        return N.device_view(address, self.shape)

    @property
    def x(self) -> torch.Tensor:
        return self.view(N.lib().pt_session_x(self.handle))

    @property
    def h(self) -> torch.Tensor:
        return self.view(N.lib().pt_session_h(self.handle))

    def buffer(self, which: int) -> torch.Tensor | None:
        addr = N.lib().pt_session_buffer(self.handle, which)
        return None if not addr else self.view(addr)

    def bad_iteration(self) -> int | None:
        t = N.device_view(N.lib().pt_session_bad_iter(self.handle), (1,), torch.int64)
        v = int(t.item())
        return None if v == INT64_MAX else v


@dataclass
class IterateState:
    """Loop state (:108-125).  x, h and the estimator/prox state live in the
    native session; the views below alias its device buffers."""

    session: _Session
    partition: SubsetPartition | None
    rng_subset: np.random.Generator
    rng_theta: np.random.Generator
    rng_refresh: np.random.Generator
    svrg_period: int | None = None
    svrg_probability: float | None = None
    iterations_since_refresh: int = 0
    k: int = 0
    data_passes: float = 0.0
    prox_calls: int = 0
    denoiser_calls: int = 0
    work_seconds: float = 0.0
    zslab: tuple | None = None  # (z0, z1, Z) when this rank holds a z-slab
    rowslab: tuple | None = None  # (r0, r1, H) when this rank holds image rows
    sharded: bool = False  # attached to a multi-rank communicator (any layout)

    @property
    def x(self) -> torch.Tensor:
        return self.session.x

    def full_x(self) -> torch.Tensor:
        """The whole iterate (a z-slab / row-slab rank gathers the other slabs)."""
        from . import distributed as _dist
        if self.zslab is not None:
            return _dist.gather_zslabs(self.session.x, self.zslab[2])
        if self.rowslab is not None:
            return _dist.gather_rowslabs(self.session.x, self.rowslab[2])
        return self.session.x

    @property
    def h(self) -> torch.Tensor:
        return self.session.h

    @property
    def saga(self):
        t = self.session.buffer(3)
        if t is None:
            return None
        n = self.partition.n_subsets
        table = N.device_view(N.lib().pt_session_buffer(self.session.handle, 3),
                              (n,) + tuple(self.session.shape))
        return est.SagaState(table=table, running_sum=self.session.buffer(2))

    @property
    def svrg(self):
        snap = self.session.buffer(0)
        if snap is None:
            return None
        return est.SvrgState(snapshot=snap, full_grad=self.session.buffer(1),
                             iterations_since_refresh=self.iterations_since_refresh,
                             refresh_period=self.svrg_period,
                             refresh_probability=self.svrg_probability)

    @property
    def tv_warm(self):
        p = self.session.buffer(4)
        if p is None or self.prox_calls == 0:
            return None
        return TvDualState(p=p, q=self.session.buffer(5), weight=float("nan"),
                           w=self.session.buffer(6))


@dataclass
class RunRecord:
    """Per-logging-event rows plus the final iterate (:128-156)."""

    rows: list = field(default_factory=list)
    iterations: list = field(default_factory=list)
    image: torch.Tensor | None = None

    def column(self, name: str) -> np.ndarray:
        j = RUN_COLUMNS.index(name)
        return np.array([math.nan if r[j] is None else float(r[j]) for r in self.rows])

    @property
    def final_rel_err(self) -> float:
        return float(self.rows[-1][RUN_COLUMNS.index("rel_err")]) if self.rows else math.nan

    def to_csv(self, path) -> None:
        with open(path, "w", encoding="utf-8") as handle:
            handle.write(",".join(RUN_COLUMNS) + "\n")
            for row in self.rows:
                handle.write(",".join("" if v is None else repr(float(v))
                                      if isinstance(v, float) else str(v)
                                      for v in row) + "\n")


def _init_state(config: SolverConfig, problem: TomoProblem, x0, stream=None,
                data_parallel: bool = False, zslab: tuple | None = None,
                rowslab: tuple | None = None, kind: str | None = None) -> IterateState:
    """solvers.py:159-186: x0 (or zeros), h = 0, three PCG64 streams, the
    staggered partition, SAGA zeros, SVRG initial snapshot (+1 pass).

    data_parallel: shard the angles over the torch.distributed ranks (one GPU
    each; the library's own NCCL communicator, see distributed.py); with
    `zslab` = (z0, z1, Z) / `rowslab` = (r0, r1, H) the problem is this
    rank's z-slab / image rows instead."""
    shape = problem.projector.shape
    if x0 is not None and tuple(x0.shape) != tuple(shape):
        raise ValueError(f"x0 shape {tuple(x0.shape)} does not match grid {shape}")
    streams = np.random.SeedSequence(config.seed).spawn(3)
    partition = None
    if config.estimator != "full":
        partition = build_staggered_partition(problem.projector.geometry.n_angles,
                                              config.n_subsets)
    stream = stream if stream is not None else torch.cuda.current_stream()
    session = _Session(config, problem, x0, stream, kind)
    if zslab is not None:
        from . import distributed as _dist
        _dist.attach_zslab(session, zslab[0], zslab[2])
    elif rowslab is not None:
        from . import distributed as _dist
        _dist.attach_rows(session, rowslab[0], rowslab[2])
    elif data_parallel:
        from . import distributed as _dist
        _dist.attach(session)
    state = IterateState(session=session, partition=partition,
                         rng_subset=np.random.default_rng(streams[0]),
                         rng_theta=np.random.default_rng(streams[1]),
                         rng_refresh=np.random.default_rng(streams[2]), zslab=zslab,
                         rowslab=rowslab, sharded=_multi_rank(data_parallel or zslab is not None
                                                              or rowslab is not None))
    if kind == "fista":
        session.init()  # y = x0, t = 1 (solvers.py:378)
    if config.estimator in ("svrg", "lsvrg"):
        if config.estimator == "svrg":
            state.svrg_period = config.n_subsets
        else:
            state.svrg_probability = 1.0 / config.n_subsets
        session.init()
        state.data_passes += 1.0
    return state


def _draw_one(state: IterateState, config: SolverConfig):
    """The reference's per-step draws and pass charge (:189-214,238)."""
    kind = config.estimator
    refresh = False
    i = 0
    if kind == "full":
        passes = 1.0
    else:
        n = state.partition.n_subsets
        if kind in ("sgd", "saga"):
            i = int(state.rng_subset.integers(n))
            passes = 1.0 / n
        else:
            passes = 0.0
            if state.svrg_period is not None:
                refresh = state.iterations_since_refresh >= state.svrg_period
            elif state.svrg_probability >= 1.0:
                refresh = True
            else:
                refresh = bool(state.rng_refresh.random() < state.svrg_probability)
            if refresh:
                state.iterations_since_refresh = 0
                passes += 1.0
            i = int(state.rng_subset.integers(n))
            state.iterations_since_refresh += 1
            passes = passes + 2.0 / n
    p = config.skip_probability
    theta = True if p >= 1.0 else bool(state.rng_theta.random() < p)
    return i, theta, refresh, passes


def _plan_segment(state: IterateState, config: SolverConfig, last_floor: int,
                  max_steps: int | None = None):
    """Steps up to and including the next log event (pass-floor crossing or
    exhaustion, :314-318).  Subset and skip draws are vectorised -- a vector
    draw consumes a PCG64 stream exactly like the same number of scalar draws
    (tests/test_host.py pins this against the reference)."""
    kind = config.estimator
    if kind == "lsvrg":
        subs, thetas, refr = [], [], []
        passes = state.data_passes
        while True:
            i, th, rf, ch = _draw_one(state, config)
            subs.append(i); thetas.append(th); refr.append(rf)
            passes += ch
            exhausted = passes >= config.max_data_passes - 1e-9
            crossed = math.floor(passes + 1e-12) > last_floor
            if crossed or exhausted or (max_steps and len(subs) >= max_steps):
                break
        return (np.array(subs), np.array(thetas), np.array(refr), passes,
                exhausted)
    n = state.partition.n_subsets if state.partition else 1
    passes = state.data_passes
    since = state.iterations_since_refresh
    charges, refr = [], []
    while True:
        rf = False
        if kind == "full":
            ch = 1.0
        elif kind in ("sgd", "saga"):
            ch = 1.0 / n
        else:
            c = 0.0
            if since >= state.svrg_period:
                rf = True
                since = 0
                c += 1.0
            since += 1
            ch = c + 2.0 / n
        passes += ch
        refr.append(rf)
        charges.append(ch)
        exhausted = passes >= config.max_data_passes - 1e-9
        crossed = math.floor(passes + 1e-12) > last_floor
        if crossed or exhausted or (max_steps and len(refr) >= max_steps):
            break
    L = len(refr)
    state.iterations_since_refresh = since
    subs = (state.rng_subset.integers(n, size=L) if kind != "full"
            else np.zeros(L, dtype=np.int64))
    p = config.skip_probability
    thetas = (np.ones(L, dtype=bool) if p >= 1.0 else state.rng_theta.random(L) < p)
    return subs, thetas, np.array(refr), passes, exhausted


def proxskip_step(state: IterateState, config: SolverConfig, problem: TomoProblem) -> IterateState:
    """One iteration of the skip-capable loop (:230-254), on the device."""
    i, theta, refresh, passes = _draw_one(state, config)
    state.session.run(np.array([i]), np.array([theta]), np.array([refresh]), state.k)
    bad = _bad_iteration(state)
    if bad is not None:
        raise DivergenceError(bad, config.gamma)
    if theta:
        state.prox_calls += 1
    state.k += 1
    state.data_passes += passes
    return state


def composite_objective(x, problem: TomoProblem) -> float:
    """0.5 ||A x - b||^2 + alpha TV(x) (:271-277): fused forward + residual +
    sum of squares on the device, then the TV reduction."""
    plan = problem.projector.plan
    xd = as_device(x)
    y = torch.empty(plan.sino_shape(problem.projector.geometry.n_angles), device="cuda",
                    dtype=torch.float32)
    sq = torch.empty(1, device="cuda", dtype=torch.float64)
    plan.forward_into(xd, y, None, data=problem.device_data(), sumsq=sq)
    value = 0.5 * float(sq.item())
    if problem.tv is not None:
        value += problem.tv.alpha * tv_value(xd)
    return value


def _metrics_row(passes, wall, x, reference, ground_truth, prox_calls, problem,
                 record_objective):
    rel = psnr_val = ssim_val = obj = None
    if reference is not None:
        rel = _relative_error_sq(x, reference)
    if ground_truth is not None:
        gt = as_device(ground_truth)
        rng_val = float(gt.max() - gt.min())
        psnr_val = _psnr(x, gt, rng_val if rng_val > 0 else 1.0)
        ssim_val = _ssim(x, gt)
    if record_objective:
        obj = composite_objective(x, problem)
    return (passes, wall, rel, psnr_val, ssim_val, prox_calls, obj)


def run(config: SolverConfig, problem: TomoProblem, x0=None, reference=None,
        ground_truth=None, record_objective: bool = False, stream=None,
        data_parallel: bool = False, decomposition: str = "sectors") -> RunRecord:
    """Run the skip-capable loop until tolerance or budget exhaustion (:327-336).

    Rows are logged at every data-pass boundary exactly as :280-324; the
    iterations between two rows are one native segment.  The host syncs only
    at rows that need a metric (or for a time budget) and at the end.
    data_parallel=True shards the work over the torch.distributed ranks (every
    rank calls run with the same arguments): the projection angles
    (decomposition "sectors", default: image and prox replicated) or the image
    rows ("rows") of a 2D problem, the
    z-slabs of a slice-stacked 3D one (the returned image is the gathered
    image / volume on every rank)."""
    return _run(config, problem, x0, reference, ground_truth, record_objective, stream,
                data_parallel, decomposition)


def _run(config, problem, x0, reference, ground_truth, record_objective, stream,
         data_parallel, decomposition, kind: str | None = None) -> RunRecord:
    if decomposition not in ("rows", "sectors"):
        raise ValueError("decomposition must be 'rows' or 'sectors'")
    if kind == "fista" and data_parallel and decomposition == "rows":
        raise ValueError("FISTA shards over angle sectors only")
    stream = stream if stream is not None else torch.cuda.current_stream()
    work, zs, rs = problem, None, None
    if (data_parallel and decomposition == "rows"
            and getattr(problem.projector, "n_slices", 1) == 1):
        import torch.distributed as dist
        from . import distributed as _dist
        H = problem.projector.height
        r0, r1 = _dist.rowslab_bounds(H, dist.get_rank(), dist.get_world_size())
        work, rs = _dist.rowslab_problem(problem, r0, r1), (r0, r1, H)
        if x0 is not None:
            x0 = as_device(x0)[r0:r1].contiguous()
    if data_parallel and getattr(problem.projector, "n_slices", 1) > 1:
        import torch.distributed as dist
        from . import distributed as _dist
        Z = problem.projector.n_slices
        z0, z1 = _dist.zslab_bounds(Z, dist.get_rank(), dist.get_world_size())
        work, zs = _dist.zslab_problem(problem, z0, z1), (z0, z1, Z)
        if x0 is not None:
            x0 = as_device(x0)[z0:z1].contiguous().reshape(work.projector.shape)
    with torch.cuda.stream(stream):
        state = _init_state(config, work, x0, stream, data_parallel=data_parallel, zslab=zs,
                            rowslab=rs, kind=kind)
        return _run_loop(state, config, problem, reference, ground_truth, record_objective,
                         stream)


def _run_loop(state: IterateState, config, problem, reference, ground_truth,
              record_objective, stream) -> RunRecord:
    record = RunRecord()
    need_metrics = reference is not None or ground_truth is not None or record_objective
    pending = []  # (row index, event-end index) for deferred wall time
    events = [torch.cuda.Event(enable_timing=True)]
    events[0].record(stream)

    def log_row(wall):
        x = state.full_x()
        row = _metrics_row(state.data_passes, wall, x, reference, ground_truth,
                           state.prox_calls, problem, record_objective)
        record.rows.append(row)
        record.iterations.append(state.k)
        return row

    def satisfied(row):
        rel = row[RUN_COLUMNS.index("rel_err")]
        return config.tolerance is not None and rel is not None and rel < config.tolerance

    row = log_row(0.0)
    if satisfied(row):
        record.image = state.full_x().clone()
        return record
    last_floor = math.floor(state.data_passes + 1e-12)
    budget = config.time_budget
    if not need_metrics and budget is None:
        # Nothing needs a value before the end: the draws are data independent,
        # so segments are planned on the host and enqueued in batches of 1, 2,
        # 4, ... segments (one native call each, an event recorded at each log
        # row): the device starts after the first segment is planned and the
        # rest is planned while it runs.
        row_events = []
        pending, marks = [], []
        n_total = n_sent = 0
        batch = 1

        def flush():
            nonlocal pending, marks, n_sent, batch
            evs = [torch.cuda.Event(enable_timing=True) for _ in marks]
            for ev in evs:
                ev.record(stream)  # materialise the handles; the native call re-records them
            state.session.run_marked(np.concatenate([p[0] for p in pending]),
                                     np.concatenate([p[1] for p in pending]),
                                     np.concatenate([p[2] for p in pending]),
                                     state.k + n_sent, [m - n_sent for m in marks], evs)
            row_events.extend(evs)
            n_sent = n_total
            pending, marks = [], []
            batch *= 2

        while True:
            subs, thetas, refr, passes, exhausted = _plan_segment(state, config, last_floor)
            pending.append((subs, thetas, refr))
            n_total += len(subs)
            state.prox_calls += int(np.count_nonzero(thetas))
            state.data_passes = passes
            marks.append(n_total)
            last_floor = math.floor(state.data_passes + 1e-12)
            record.rows.append((state.data_passes, None, None, None, None, state.prox_calls,
                                None))
            record.iterations.append(state.k + n_total)
            if exhausted or len(pending) >= batch:
                flush()
            if exhausted:
                break
        state.k += n_total
        stream.synchronize()
        for ri, ev in enumerate(row_events, start=1):
            r = record.rows[ri]
            record.rows[ri] = (r[0], events[0].elapsed_time(ev) / 1e3) + tuple(r[2:])
        state.work_seconds = record.rows[-1][1]
        bad = _bad_iteration(state)
        if bad is not None:
            raise _diverged(bad, config, record)
        record.image = state.full_x().clone()
        record.state = state
        return record
    while True:
        subs, thetas, refr, passes, exhausted = _plan_segment(
            state, config, last_floor, max_steps=1 if budget is not None else None)
        state.session.run(subs, thetas, refr, state.k)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        events.append(ev)
        state.k += len(subs)
        state.prox_calls += int(np.count_nonzero(thetas))
        state.data_passes = passes
        if budget is not None or need_metrics:
            ev.synchronize()
            state.work_seconds = (state.work_seconds
                                  + events[-2].elapsed_time(events[-1]) / 1e3)
            if budget is not None:
                exhausted = exhausted or state.work_seconds >= budget
            bad = _bad_iteration(state)
            if bad is not None:
                raise _diverged(bad, config, record)
        crossed = math.floor(state.data_passes + 1e-12) > last_floor
        if crossed or exhausted:
            last_floor = math.floor(state.data_passes + 1e-12)
            if need_metrics or budget is not None:
                row = log_row(state.work_seconds)
            else:
                row = (state.data_passes, None, None, None, None, state.prox_calls, None)
                record.rows.append(row)
                record.iterations.append(state.k)
                pending.append((len(record.rows) - 1, len(events) - 1))
            if satisfied(row) or exhausted:
                break
    if pending:
        # wall_seconds of deferred rows: cumulative device time of segments
        stream.synchronize()
        cum = [0.0]
        for j in range(1, len(events)):
            cum.append(cum[-1] + events[j - 1].elapsed_time(events[j]) / 1e3)
        for ri, ei in pending:
            r = record.rows[ri]
            record.rows[ri] = (r[0], cum[ei]) + tuple(r[2:])
        state.work_seconds = cum[-1]
    bad = _bad_iteration(state)
    if bad is not None:
        raise _diverged(bad, config, record)
    record.image = state.full_x().clone()
    record.state = state
    return record


def _multi_rank(attached: bool) -> bool:
    if not attached:
        return False
    import torch.distributed as dist
    return dist.is_initialized() and dist.get_world_size() > 1


def _bad_iteration(state: IterateState) -> int | None:
    """First non-finite iteration; on several ranks the minimum over ranks
    (each rank checks the pixels it computed: its slab, or its rows of a
    sharded prox), so every rank raises together."""
    bad = state.session.bad_iteration()
    if not state.sharded:
        return bad
    import torch.distributed as dist
    t = torch.tensor([INT64_MAX if bad is None else bad], device="cuda", dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    v = int(t.item())
    return None if v == INT64_MAX else v


def _diverged(bad: int, config: SolverConfig, record: RunRecord) -> DivergenceError:
    keep = [j for j, it in enumerate(record.iterations) if it <= bad]
    record.rows = [record.rows[j] for j in keep]
    record.iterations = [record.iterations[j] for j in keep]
    record.image = None
    return DivergenceError(bad, config.gamma, record)


# ----------------------------------------------------------------------------
# Deterministic reference solvers (solvers.py:339-392) built from the same
# native operators.  They keep the reference's loop and logging semantics.
# ----------------------------------------------------------------------------

def _full_gradient_config(config: SolverConfig) -> SolverConfig:
    """The reference's ISTA / FISTA keep only these fields of the caller's
    config (solvers.py:346-350,371-375): full gradient, no skipping."""
    return SolverConfig(gamma=config.gamma, max_data_passes=config.max_data_passes,
                        tolerance=config.tolerance, time_budget=config.time_budget,
                        seed=config.seed)


def run_ista(config: SolverConfig, problem: TomoProblem, x0=None, reference=None,
             ground_truth=None, record_objective: bool = False, stream=None,
             data_parallel: bool = False) -> RunRecord:
    """x+ = prox_gamma(x - gamma grad f(x)) (:339-364), on the native executor:
    ProxSkip with the full-gradient estimator at p = 1 is exactly this step
    (hcoef = gamma - gamma/p = 0, so h never reaches x), with the same pass
    accounting (1 per iteration) and rows."""
    return _run(_full_gradient_config(config), problem, x0, reference, ground_truth,
                record_objective, stream, data_parallel, "sectors")


def run_fista(config: SolverConfig, problem: TomoProblem, x0=None, reference=None,
              ground_truth=None, record_objective: bool = False, stream=None,
              data_parallel: bool = False) -> RunRecord:
    """Accelerated variant, prox every iteration (:367-392), on the native
    executor: per step one fused full-gradient pass at the momentum point y
    (forward - b, gather + y - gamma g), the TV prox, and one momentum kernel
    (x+ finite check, y = x+ + beta_k (x+ - x)); t_k is kept in float64 on the
    host side of the session.  No host synchronisation between log rows."""
    return _run(_full_gradient_config(config), problem, x0, reference, ground_truth,
                record_objective, stream, data_parallel, "sectors", kind="fista")


def run_pdhg_reference(problem: TomoProblem, n_iterations: int, snapshot_at: int | None = None):
    """High-accuracy reference by diagonally preconditioned primal-dual
    iterations on the saddle form (solvers.py:395-455), on the device.

    Per iteration: the forward with the data subtraction fused (A xbar - b),
    the dual sinogram step, the gather adjoint, the TV dual step and the
    primal step (pdhg.cu).  Returns the final iterate, or (final, snapshot)
    when ``snapshot_at`` is given; device float32 tensors.  A non-finite
    iterate raises DivergenceError(first bad iteration, max tau)."""
    if n_iterations < 1:
        raise ValueError("n_iterations must be >= 1")
    if problem.denoiser is not None:
        raise ValueError("reference solver needs an explicit objective, not a denoiser")
    projector = problem.projector
    if getattr(projector, "n_slices", 1) != 1:
        raise ValueError("the PDHG reference is 2D (solvers.py:395-455)")
    data = problem.device_data()
    alpha = problem.tv.alpha if problem.tv is not None else 0.0
    nonneg = problem.tv.nonneg if problem.tv is not None else False
    H, W = projector.shape
    plan = projector.plan
    lib = N.lib()
    stream = N.stream_handle()
    ones = torch.ones((H, W), device="cuda")
    row_sums = torch.empty_like(data)
    plan.forward_into(ones, row_sums)
    sigma_a = torch.where(row_sums > 0, 1.0 / row_sums, torch.zeros_like(row_sums)).contiguous()
    col_sums = torch.empty((H, W), device="cuda")
    plan.adjoint_into(torch.ones_like(data), col_sums)
    if alpha > 0.0:
        diff_cols = torch.zeros((H, W), device="cuda")
        diff_cols[:-1, :] += 1.0
        diff_cols[1:, :] += 1.0
        diff_cols[:, :-1] += 1.0
        diff_cols[:, 1:] += 1.0
        col_sums = col_sums + diff_cols
    tau = (1.0 / torch.clamp(col_sums, min=1e-12)).contiguous()
    sigma_d = 0.5
    x = torch.zeros((H, W), device="cuda")
    x_bar = torch.zeros_like(x)
    y = torch.zeros_like(data)
    resid = torch.empty_like(data)
    ascent = torch.empty_like(x)
    zv = torch.zeros_like(x) if alpha > 0.0 else None
    zh = torch.zeros_like(x) if alpha > 0.0 else None
    bad = torch.full((1,), 2 ** 62, device="cuda", dtype=torch.int64)
    snapshot = None
    for it in range(1, n_iterations + 1):
        plan.forward_into(x_bar, resid, data=data)
        N.check(lib.pt_pdhg_dual_sino(N.ptr(y), N.ptr(resid), N.ptr(sigma_a), y.numel(),
                                      stream), "pdhg")
        plan.adjoint_into(y, ascent)
        if alpha > 0.0:
            N.check(lib.pt_pdhg_dual_tv(N.ptr(x_bar), N.ptr(zv), N.ptr(zh), 1, H, W, sigma_d,
                                        float(alpha), stream), "pdhg")
        N.check(lib.pt_pdhg_primal(N.ptr(x), N.ptr(x_bar), N.ptr(ascent), N.ptr(zv), N.ptr(zh),
                                   N.ptr(tau), 1, H, W, int(bool(nonneg)), it, N.ptr(bad),
                                   stream), "pdhg")
        if snapshot_at is not None and it == snapshot_at:
            snapshot = x.clone()
    first_bad = int(bad.item())
    if first_bad < 2 ** 62:
        raise DivergenceError(first_bad, float(tau.max()))
    if snapshot_at is not None:
        return x, snapshot
    return x


def optimal_p(mu: float, lipschitz: float) -> float:
    """sqrt(mu / L) clamped into (0, 1] (:458-465)."""
    if mu <= 0.0 or lipschitz <= 0.0:
        raise ValueError("mu and L must be positive")
    if mu > lipschitz:
        raise ValueError("mu cannot exceed L")
    return min(1.0, math.sqrt(mu / lipschitz))


def default_gamma(estimator: str, lipschitz: float) -> float:
    """1.99/L full, 1/(3L) saga, 1/L otherwise (:468-479)."""
    if lipschitz <= 0.0:
        raise ValueError("L must be positive")
    if estimator == "full":
        return 1.99 / lipschitz
    if estimator == "saga":
        return 1.0 / (3.0 * lipschitz)
    if estimator in ("sgd", "svrg", "lsvrg"):
        return 1.0 / lipschitz
    raise ValueError(f"unknown estimator {estimator!r}")


def fista_gamma(lipschitz: float) -> float:
    if lipschitz <= 0.0:
        raise ValueError("L must be positive")
    return 1.0 / lipschitz
