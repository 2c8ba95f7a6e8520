#!/usr/bin/env python
"""Benchmark: ProxSkip-SVRG epochs/s of the B200-native hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One JSON line (rank 0).  Workload: BASELINE.json configs[2] by default --
2048^2 image, 1800 angles x 2900 bins, 60 interleaved subsets, ProxSkip-SVRG
(p = 0.05, gamma = 1/L), FGP-TV 100 inner iterations -- the SVRG config the
metric names, and the one that shards over 1/2/4/8 GPUs.  A "step" is one
epoch (one snapshot full gradient + N ProxSkip iterations),
continuing one trajectory: W warm-up epochs, then K timed epochs.

value  : epochs/s of the whole job (device time, CUDA events on the solver
         stream, barrier + synchronize on both sides, max over ranks), the
         problem already resident in HBM;
e2e    : the same metric through the public API ``run(config, problem)`` with
         the sinogram in pinned HOST memory (H2D inside the timed region) and
         the reconstruction read back to the host (D2H inside);
roofline: the dominant kernel of the timed region (live CUDA-event timing of
         each launch category) against SURVEY.md 8d's algorithmic bytes;
cpu_baseline: the float64 oracle port (oracle/, all host threads) on a
         bounded sample of the same workload.
``--impl reference`` times that CPU port alone as the reference arm.
"""

from __future__ import annotations

import argparse
import glob
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=["c0", "c1", "c2", "c3"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--decomposition", default="rows", choices=["rows", "sectors"],
                    help="2D multi-GPU layout: image rows (default) or angle sectors")
    ap.add_argument("--dp-one-rank", action="store_true",
                    help="test hook: run the multi-GPU data path (NCCL process group, sharded "
                         "session) with a single rank")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def l2_note(cfg):
    """Touched bytes per epoch vs the 126 MB L2 (the timing rule's flush question):
    image-sized state (x, h, x_snap, full gradient, FGP work planes, SAGA table),
    the sinogram and residuals, and the band partials of the snapshot's forward."""
    n = cfg.size * cfg.size * cfg.depth
    rays = cfg.n_angles * cfg.n_bins * cfg.depth
    bands = -(-cfg.size // (64 if cfg.size >= 512 else 32))
    planes = 6 + 8 + (cfg.n_subsets if cfg.estimator == "saga" else 0)
    ws = 4 * (n * planes + 2 * rays)
    if cfg.estimator in ("svrg", "lsvrg"):
        ws += 4 * bands * rays
    if ws > 126e6:
        return f"working set ~{ws / 1e6:.0f} MB > L2 (126 MB); no flush"
    return (f"working set ~{ws / 1e6:.0f} MB < L2 (126 MB); no flush: the solver state stays "
            f"L2-resident across steps in any run of this size")


def workload_name(cfg):
    dim = f"{cfg.size}^3" if cfg.depth > 1 else f"{cfg.size}^2"
    return (f"{cfg.name}: {dim}, {cfg.n_angles} angles x {cfg.n_bins} bins, N={cfg.n_subsets} "
            f"ProxSkip-{cfg.estimator.upper()} p={cfg.p}, FGP-TV {cfg.fgp_inner}, "
            f"{cfg.epochs}-epoch run")


# --------------------------------------------------------------------------
# CPU: the oracle port (reference arm and cpu_baseline)
# --------------------------------------------------------------------------

def cpu_problem(cfg, b=None):
    """Same inputs as the GPU arm on the host in float64 (phantom law, noise,
    alpha); `b` may be handed over from the GPU arm (setup, untimed)."""
    import oracle as O
    from paper_2602_09527_b200 import problems
    from paper_2602_09527_b200.geometry import ParallelGeometry
    O.set_mode("fast")
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = O.OracleProjector(g, cfg.size, cfg.size, cfg.depth)
    if b is None:
        x_true = problems.phantom_for(cfg).astype(np.float64)
        b = problems.add_noise(proj.forward(x_true), cfg.noise, cfg.noise_seed)
    alpha = problems.alpha_from_backprojection(float(np.abs(proj.adjoint(b)).max()),
                                                cfg.n_pixels)
    return O, proj, b, alpha


def cpu_epochs_per_second(cfg, seconds, gamma, alpha, b):
    """Epochs/s of the float64 oracle restatement (all host threads) on a
    bounded sample: one snapshot full gradient, then ProxSkip iterations with
    the reference's draws for ~`seconds` (loop timer as solvers.py:304-313);
    epoch time = snapshot + N x mean iteration time (prox calls included)."""
    import oracle as O
    from oracle import solver as S
    from paper_2602_09527_b200.geometry import ParallelGeometry
    O.set_mode("fast")
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = O.OracleProjector(g, cfg.size, cfg.size, cfg.depth)
    x0 = np.zeros(proj.shape)
    t0 = time.perf_counter()
    proj.adjoint(proj.forward(x0) - b)  # one snapshot full gradient (estimators.py:40-48)
    t_snap = time.perf_counter() - t0
    r = S.run_proxskip(proj, b, gamma=gamma, p=cfg.p, estimator=cfg.estimator,
                       n_subsets=cfg.n_subsets, max_data_passes=cfg.max_data_passes,
                       seed=cfg.solver_seed, tv_alpha=alpha, tv_inner=cfg.fgp_inner,
                       max_seconds=seconds, max_iterations=cfg.n_subsets)
    per_iter = r.work_seconds / max(1, r.k)
    snap = t_snap if cfg.estimator in ("svrg", "lsvrg") else 0.0
    epoch_s = snap + cfg.n_subsets * per_iter
    return 1.0 / epoch_s, r.k, r.work_seconds + t_snap, r.prox_calls, O.nthreads()


def reference_arm(args, cfg, rank, world):
    if rank != 0:
        return 0
    from paper_2602_09527_b200 import problems  # noqa: F401
    from oracle import solver as S
    prob = cpu_problem(cfg)
    O, proj, b, alpha = prob
    gamma = 1.0 / O.operator_norm_sq(proj.geometry, cfg.size, cfg.size, 5, cfg.power_seed)
    # one "step" = a bounded slice of the solve: N/6 iterations (snapshot
    # refreshes and prox calls included as they fall), one continuing trajectory
    per_step = max(1, cfg.n_subsets // 6)
    total_iters = (args.warmup + args.steps) * per_step
    rw = S.run_proxskip(proj, b, gamma=gamma, p=cfg.p, estimator=cfg.estimator,
                        n_subsets=cfg.n_subsets, max_data_passes=cfg.max_data_passes,
                        seed=cfg.solver_seed, tv_alpha=alpha, tv_inner=cfg.fgp_inner,
                        max_iterations=total_iters)
    w_iters = min(args.warmup * per_step, rw.k)
    t_w = rw.cum_seconds[w_iters - 1] if w_iters else 0.0
    timed_iters = rw.k - w_iters
    timed_s = rw.work_seconds - t_w
    value = (timed_iters / cfg.n_subsets) / timed_s
    line = {
        "impl": "reference", "metric": "ProxSkip-SVRG epochs/s", "value": value,
        "unit": "epochs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * timed_s / max(1, args.steps), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(cfg), "step": f"{per_step} ProxSkip iterations",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "epochs/s", "cores": O.nthreads(), "kind": "port",
                         "sample": f"{timed_iters} iterations ({timed_iters / cfg.n_subsets:.3f} "
                                   f"epochs) of the float64 oracle restatement"},
        "e2e": {"value": value, "unit": "epochs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"pt_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            # timed region shorter than nvidia-smi's start-up (configs 0 / 1):
            # one query right after it, the clocks still at their loaded state
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=10).stdout
                rows = [[p.strip() for p in ln.split(",")] for ln in out.splitlines()
                        if len(ln.split(",")) >= 9]
            except Exception:
                rows = []
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def build_gpu_problem(cfg, torch):
    """Synthetic BASELINE problem on the device: phantom (host law), b = A x
    (device) + host noise, alpha from A^T b, L by 50 power iterations."""
    from paper_2602_09527_b200 import (ParallelGeometry, Projector, TomoProblem, TvProxConfig,
                                       default_gamma, problems)
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = Projector(g, cfg.size, cfg.size, cfg.depth)
    x_true = problems.phantom_for(cfg)
    clean = proj.forward(x_true).double().cpu().numpy()
    b = problems.add_noise(clean, cfg.noise, cfg.noise_seed)
    b_host = torch.from_numpy(b.astype(np.float32)).pin_memory()
    b_dev = b_host.to("cuda")
    alpha = problems.alpha_from_backprojection(float(proj.adjoint(b_dev).abs().max()),
                                               cfg.n_pixels)
    lip = proj.norm_sq(cfg.power_iterations, cfg.power_seed)
    gamma = default_gamma(cfg.estimator, lip)
    tv = TvProxConfig(alpha=alpha, inner_iterations=cfg.fgp_inner)
    return proj, b_host, b_dev, TomoProblem(proj, b_dev, tv=tv), gamma, alpha, lip


def algorithmic_bytes(cfg, proj, state):
    """SURVEY.md 8d per-launch algorithmic bytes of each launch category."""
    depth = getattr(proj, "n_slices", 1)  # this rank's planes (z-slab) or the volume
    n_px = proj.width * proj.height * depth  # this rank's pixels (row / z slab or all)
    plan = proj.plan
    part = state.partition
    sub0 = part.subsets[0] if part else None
    nnz = plan.nnz(sub0) if sub0 else plan.nnz(None)
    rays = (len(sub0) if sub0 else cfg.n_angles) * cfg.n_bins * depth
    e = 4 if cfg.estimator in ("svrg", "lsvrg") else (7 if cfg.estimator == "saga" else 3)
    return {
        "fwd_band": 4 * nnz + 4 * rays,
        "gather_step": 4 * nnz + 4 * n_px * e,
        "fgp_call": (40 if cfg.depth > 1 else 28) * n_px * cfg.fgp_inner + 28 * n_px,
        "fwd_reduce": None, "snapshot": None, "other": None,
    }, nnz


def ncu_traffic(kernel_key):
    """dram bytes per launch of the top kernel from the committed ncu capture."""
    best = None
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "*ncu_traffic*.json"))):
        try:
            with open(path) as fh:
                d = json.load(fh)
            if kernel_key in d:
                best = d[kernel_key]
        except Exception:
            pass
    return best


def gpu_arm(args, cfg, rank, world, local):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dp = world > 1 or args.dp_one_rank  # the multi-GPU data path
    if dp:
        if "RANK" not in os.environ:  # --dp-one-rank without torchrun: a one-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2602_09527_b200 import SolverConfig, TomoProblem, run
    from paper_2602_09527_b200 import _native as N
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200.solvers import _init_state, _plan_segment

    proj, b_host, b_dev, problem, gamma, alpha, lip = build_gpu_problem(cfg, torch)
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=1e18, seed=cfg.solver_seed)
    stream = torch.cuda.Stream()
    # multi-GPU: image rows or angle sectors (2D), z-slabs (slice-stacked 3D);
    # SURVEY.md 8e, DESIGN.md "Multi-GPU"
    zs, rs, work = None, None, problem
    if dp and cfg.depth > 1:
        z0, z1 = D.zslab_bounds(cfg.depth, rank, world)
        zs, work = (z0, z1, cfg.depth), D.zslab_problem(problem, z0, z1)
    elif dp and args.decomposition == "rows":
        r0, r1 = D.rowslab_bounds(cfg.size, rank, world)
        rs, work = (r0, r1, cfg.size), D.rowslab_problem(problem, r0, r1)
    with torch.cuda.stream(stream):
        state = _init_state(scfg, work, None, stream, zslab=zs, rowslab=rs)
    if dp and zs is None and rs is None:
        D.attach(state.session)
        # re-initialise the snapshot with the sharded full gradient
        state.session.init()
    sess = state.session

    def run_epochs(n_epochs):
        """n epochs = n*N iterations with the reference's draws."""
        n_steps = n_epochs * cfg.n_subsets
        scfg_local = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                                  estimator=cfg.estimator,
                                  max_data_passes=state.data_passes + 1e12, seed=cfg.solver_seed)
        subs, thetas, refr, passes, _ = _plan_segment(state, scfg_local, 1 << 62,
                                                      max_steps=n_steps)
        sess.run(subs, thetas, refr, state.k)
        state.k += len(subs)
        state.data_passes = passes
        state.prox_calls += int(np.count_nonzero(thetas))
        return len(subs), int(np.count_nonzero(thetas))

    def barrier():
        if dp:
            dist.barrier()

    # warm-up
    run_epochs(args.warmup)
    stream.synchronize()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = N.launch_count()
    torch.cuda.synchronize()
    barrier()
    t_start.record(stream)
    n_iter, n_prox = run_epochs(args.steps)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = N.launch_count() - launches0
    clock_info = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    if dp:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    bad = sess.bad_iteration()
    value = args.steps / (ms / 1e3)

    # replica check across ranks
    # replicas exist only in the angle-sector layout (slab layouts own disjoint parts)
    replicas_ok = D.replicas_identical(sess.x) if (dp and zs is None and rs is None) else None

    # live per-kernel timing: a second timed pass with CUDA events per launch
    roofline = None
    kernel_times = None
    if not args.no_profile:
        N.check(N.lib().pt_session_set_profiling(sess.handle, 1))
        run_epochs(max(1, min(args.steps, 3)))
        import ctypes
        msa = (ctypes.c_double * 6)()
        cnt = (ctypes.c_int64 * 6)()
        N.check(N.lib().pt_session_profile(sess.handle, msa, cnt))
        N.check(N.lib().pt_session_set_profiling(sess.handle, 0))
        tot = sum(msa)
        kernel_times = {name: {"ms": round(msa[i], 3), "calls": int(cnt[i]),
                               "share": round(msa[i] / tot, 4) if tot else None}
                        for i, name in enumerate(N.PROF_NAMES)}
        alg, nnz = algorithmic_bytes(cfg, work.projector, state)  # per rank
        cands = [k for k in ("gather_step", "fwd_band", "fgp_call") if alg[k] and cnt[N.PROF_NAMES.index(k)]]
        top = max(cands, key=lambda k: msa[N.PROF_NAMES.index(k)])
        i = N.PROF_NAMES.index(top)
        per_launch_s = msa[i] / cnt[i] / 1e3
        achieved = alg[top] / per_launch_s / 1e9
        peak, peak_kind = peaks()
        roofline = {"bound": "hbm", "kernel": top, "achieved": round(achieved, 1), "peak": peak,
                    "unit": "GB/s", "frac": round(achieved / peak, 4),
                    "traffic": ncu_traffic(top), "peak_source": peak_kind,
                    "bytes_per_launch": alg[top], "avg_launch_us": round(per_launch_s * 1e6, 2),
                    "nnz_subset0": nnz,
                    "note": "algorithmic bytes (SURVEY.md 8d: 4 B per Joseph nonzero + epilogue "
                            "arrays); > 1 means on-chip operand reuse"}

    # end-to-end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        e2e_epochs = min(cfg.epochs, max(args.steps, 3))
        ecfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                            estimator=cfg.estimator,
                            max_data_passes=(3.0 if cfg.estimator in ("svrg", "lsvrg") else 1.0)
                            * e2e_epochs, seed=cfg.solver_seed)
        # one untimed 1-epoch solve warms the plan caches and leaves the session's
        # memory in torch's caching allocator (as in any repeated use of run()),
        # then H2D + solve + D2H are timed
        host_out = torch.empty(proj.shape, dtype=torch.float32).pin_memory()
        wcfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                            estimator=cfg.estimator,
                            max_data_passes=3.0 if cfg.estimator in ("svrg", "lsvrg") else 1.0,
                            seed=cfg.solver_seed)
        warm = run(wcfg, TomoProblem(proj, b_host, tv=problem.tv), data_parallel=dp,
                   decomposition=args.decomposition)
        del warm
        import gc
        gc.collect()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        prob_h = TomoProblem(proj, b_host, tv=problem.tv)
        rec = run(ecfg, prob_h, data_parallel=dp, decomposition=args.decomposition)
        host_out.copy_(rec.image, non_blocking=True)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        if dp:  # the job's end-to-end time is the slowest rank's
            tw = torch.tensor([wall], device="cuda", dtype=torch.float64)
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
            wall = float(tw.item())
        e2e = {"value": e2e_epochs / wall, "unit": "epochs/s",
               "h2d_bytes_per_step": int(b_host.numel() * 4 / e2e_epochs),
               "d2h_bytes_per_step": int(host_out.numel() * 4 / e2e_epochs),
               "note": f"run() over {e2e_epochs} epochs incl. session setup, initial snapshot, "
                       f"H2D of the pinned sinogram and D2H of the image (after one untimed "
                       f"1-epoch run() that warms the plan and allocator caches)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            b64 = b_host.double().numpy()
            v, k, secs, nprox, cores = cpu_epochs_per_second(cfg, args.cpu_seconds, gamma,
                                                             alpha, b64)
            cpu = {"value": v, "unit": "epochs/s", "cores": cores, "kind": "port",
                   "sample": f"1 snapshot full gradient + {k} ProxSkip-{cfg.estimator.upper()} "
                             f"iterations ({nprox} prox calls, {secs:.1f} s) of the float64 oracle "
                             f"restatement on the same problem; epoch = snapshot + N x mean "
                             f"iteration"}
        except Exception as exc:  # the baseline must not kill the bench line
            cpu = {"value": None, "unit": "epochs/s", "cores": None, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "ProxSkip-SVRG epochs/s", "value": value, "unit": "epochs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_name(cfg), "step": "1 epoch = snapshot + N iterations",
                       "epochs_timed": args.steps, "iterations_timed": n_iter,
                       "prox_calls_timed": n_prox,
                       "parallelism": ("1 GPU" if not dp else
                                       f"z-slab dp{world}" if zs else
                                       f"image-row dp{world}" if rs else
                                       f"angle-sector dp{world}"),
                       "l2": l2_note(cfg),
                       "L": lip, "gamma": gamma, "alpha": alpha},
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clock_info, "kernel_times": kernel_times,
            "finite": bad is None, "replicas_identical": replicas_ok,
        }
        print(json.dumps(line), flush=True)
    if dp:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    # stdout carries exactly one JSON line: the image sets NCCL_DEBUG=VERSION,
    # and with NCCL_DEBUG set at all the "NCCL version" banner lands on stdout
    # at communicator init (measured on the B200 image); a bare VERSION request
    # is dropped, any other debug level is the user's choice and kept
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        os.environ.pop("NCCL_DEBUG")
    from paper_2602_09527_b200 import problems
    cfg = problems.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)
    return gpu_arm(args, cfg, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
