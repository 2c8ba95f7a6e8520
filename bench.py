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
import os
import statistics
import subprocess
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2602_09527_b200._native import PROF_NAMES  # noqa: E402  (no device needed)
from paper_2602_09527_b200.problems import POWER_L  # noqa: E402


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
    ap.add_argument("--decomposition", default="sectors", choices=["sectors", "rows"],
                    help="2D multi-GPU layout: angle sectors with a replicated image "
                         "(north_star's layout, default; the TV prox sharded by rows, "
                         "PT_SECTOR_PROX=0 replicates it) or image rows")
    ap.add_argument("--dry-run", action="store_true",
                    help="test hook: form the N-rank process group (gloo, no GPU work) and "
                         "print its size; used by tests/test_bench_cli.py")
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


def bench_config(cfg):
    """The `config` object both arms print (identical, so the driver can
    compare them): the workload, the unit of the metric and the problem
    constants' provenance.  Per-arm details (what one timed step is, the
    parallelism) are top-level keys."""
    return {"workload": workload_name(cfg),
            "epoch": "1 SVRG snapshot full gradient + N ProxSkip iterations (SURVEY.md 8d)"
                     if cfg.estimator in ("svrg", "lsvrg") else "N ProxSkip iterations",
            "L": f"{cfg.power_iterations} power iterations, seed {cfg.power_seed} "
                 f"(problems.POWER_L['{cfg.name}'] = {POWER_L[cfg.name]!r})",
            "alpha": "0.01 max|A^T b| / n_pixels",
            "l2": l2_note(cfg)}


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
    """The reference's algorithm on the host (float64 oracle port, all host
    threads; the reference itself is Python/scipy and cannot run config 2:
    SURVEY.md 0).  Same problem, gamma and draws as the GPU arm; one
    continuing trajectory of which each timed step is a bounded slice of N/6
    iterations (snapshot refreshes and prox calls included as they fall);
    epochs/s = timed iterations / N / timed seconds."""
    if rank != 0:
        return 0
    from oracle import solver as S
    O, proj, b, alpha = cpu_problem(cfg)
    gamma = default_gamma_for(cfg)
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
        "config": bench_config(cfg),
        "step": f"{per_step} ProxSkip iterations of one continuing trajectory",
        "parallelism": f"{O.nthreads()} host threads (OpenMP)",
        "cpu_baseline": {"value": value, "unit": "epochs/s", "cores": O.nthreads(), "kind": "port",
                         "sample": f"{timed_iters} iterations ({timed_iters / cfg.n_subsets:.3f} "
                                   f"epochs, {rw.prox_calls} prox calls in the whole run) of "
                                   f"the float64 oracle restatement"},
        "e2e": {"value": value, "unit": "epochs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "problem": {"gamma": gamma, "alpha": alpha},
    }
    print(json.dumps(line), flush=True)
    return 0


def default_gamma_for(cfg):
    """gamma from the pinned L (problems.POWER_L) by the reference's rule
    (solvers.py:468-479)."""
    from paper_2602_09527_b200.solvers import default_gamma
    return default_gamma(cfg.estimator, POWER_L[cfg.name])


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
    (device) + host noise, alpha from A^T b; gamma from the pinned L."""
    from paper_2602_09527_b200 import (ParallelGeometry, Projector, TomoProblem, TvProxConfig,
                                       problems)
    g = ParallelGeometry.uniform(cfg.n_angles, cfg.n_bins)
    proj = Projector(g, cfg.size, cfg.size, cfg.depth)
    x_true = problems.phantom_for(cfg)
    clean = proj.forward(x_true).double().cpu().numpy()
    b = problems.add_noise(clean, cfg.noise, cfg.noise_seed)
    b_host = torch.from_numpy(b.astype(np.float32)).pin_memory()
    b_dev = b_host.to("cuda")
    alpha = problems.alpha_from_backprojection(float(proj.adjoint(b_dev).abs().max()),
                                               cfg.n_pixels)
    gamma = default_gamma_for(cfg)
    tv = TvProxConfig(alpha=alpha, inner_iterations=cfg.fgp_inner)
    return proj, b_host, b_dev, TomoProblem(proj, b_dev, tv=tv), gamma, alpha


# --------------------------------------------------------------------------
# roofline of the timed region (SURVEY.md 8d algorithmic bytes)
# --------------------------------------------------------------------------

# launch category -> (kernel, ncu kernel-name key) as in profiles/ncu_roofline_*.json
KERNEL_OF = {"fwd_band": "fwd_band_kernel", "gather": "adj_gather_kernel",
             "fgp": "fgp2d_kernel", "fgp3": "fgp3d_col3_kernel"}


def sector_prox_sharded(world):
    """Whether the sector layout's TV prox runs sharded by image rows (the
    library's rule: > 1 rank, PT_SECTOR_PROX not 0; >= 9 rows per rank holds
    for every 2D config)."""
    return world > 1 and os.environ.get("PT_SECTOR_PROX", "1") != "0"


def owned_angles(cfg, rank, world, sectors):
    if not sectors:
        return None
    return (cfg.n_angles * rank // world, cfg.n_angles * (rank + 1) // world)


def epoch_algorithmic_bytes(cfg, plan, subs, refr, n_prox, n_px, depth, own):
    """Total algorithmic bytes of the timed steps per kernel family:
    forward 4 nnz_i + 4 R_i per subset launch (+ the snapshot's all-angle
    launch per refresh), gather 4 nnz_i + 4 n_px e (SVRG step e = 4: x, h,
    grad f(x~), x-hat / x+; snapshot gather e = 1), FGP 28 (2D) / 40 (3D)
    bytes per pixel per inner iteration + 28 for the epilogue."""
    n = cfg.n_subsets

    def sel(k):
        angles = list(range(k, cfg.n_angles, n))
        if own:
            angles = [a for a in angles if own[0] <= a < own[1]]
        return angles

    nnz_sub, rays_sub = {}, {}
    for k in range(n):
        a = sel(k)
        nnz_sub[k] = plan.nnz(tuple(a)) if a else 0
        rays_sub[k] = len(a) * cfg.n_bins * depth
    all_angles = (list(range(own[0], own[1])) if own else None)
    nnz_all = plan.nnz(tuple(all_angles) if own else None)
    rays_all = (len(all_angles) if own else cfg.n_angles) * cfg.n_bins * depth
    e = 4 if cfg.estimator in ("svrg", "lsvrg") else (7 if cfg.estimator == "saga" else 3)
    fwd = gat = 0
    n_fwd = 0
    for i, rf in zip(subs, refr):
        if rf:
            fwd += 4 * nnz_all + 4 * rays_all
            gat += 4 * nnz_all + 4 * n_px
            continue  # the post-refresh step runs no projection
        fwd += 4 * nnz_sub[int(i)] + 4 * rays_sub[int(i)]
        gat += 4 * nnz_sub[int(i)] + 4 * n_px * e
        n_fwd += 1
    fgp_b = ((40 if depth > 1 else 28) * n_px * cfg.fgp_inner + 28 * n_px) * n_prox
    return {"fwd_band": fwd, "gather": gat, "fgp": fgp_b}, nnz_sub[0], n_fwd


def ncu_binding(config_name, kernel):
    """Per-launch ncu figures of `kernel` captured on THIS config (the
    newest profiles/ncu_roofline_r*.json that has the pair), else None."""
    found = None
    for path in sorted(glob.glob(os.path.join(REPO, "profiles", "ncu_roofline_r*.json"))):
        try:
            with open(path) as fh:
                d = json.load(fh)
        except Exception:
            continue
        rec = d.get(config_name, {}).get(kernel)
        if rec:
            found = dict(rec, source=os.path.relpath(path, REPO))
    return found


def roofline_record(cfg, msa, cnt, alg, peak, peak_kind):
    """Dominant kernel of the timed region (subset + snapshot launches) and its
    achieved algorithmic GB/s; binding fractions from the same config's ncu
    capture decide `bound`."""
    idx = {name: i for i, name in enumerate(PROF_NAMES)}
    ms = {"fwd_band": msa[idx["fwd_band"]] + msa[idx["snap_fwd_band"]],
          "gather": msa[idx["gather_step"]] + msa[idx["snap_gather"]],
          "fgp": msa[idx["fgp_call"]]}
    launches = {"fwd_band": cnt[idx["fwd_band"]] + cnt[idx["snap_fwd_band"]],
                "gather": cnt[idx["gather_step"]] + cnt[idx["snap_gather"]],
                "fgp": cnt[idx["fgp_call"]]}
    cands = [k for k in ms if ms[k] > 0 and alg[k]]
    if not cands:
        return None
    top = max(cands, key=lambda k: ms[k])
    achieved = alg[top] / (ms[top] / 1e3) / 1e9
    kernel = KERNEL_OF["fgp3" if (top == "fgp" and cfg.depth > 1) else top]
    if top == "fwd_band" and cfg.depth == 1 and cfg.size <= 128:
        kernel = "fwd_small_kernel"  # images <= 128^2: one-launch forward (projector.cu)
    rec = {"kernel": kernel, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "peak_source": peak_kind,
           "algorithmic_bytes_timed": int(alg[top]), "ms_timed": round(ms[top], 3),
           "calls": int(launches[top]),
           "avg_call_us": round(1e3 * ms[top] / max(1, launches[top]), 2),
           "share_of_profiled_step": None, "traffic": None, "bound": None,
           "note": "achieved = SURVEY.md 8d algorithmic bytes (one 4-byte operand per Joseph "
                   "nonzero + the arrays each kernel must touch) / CUDA-event time, summed over "
                   "the subset and snapshot launches of the profiled epochs; > 1 of HBM peak is "
                   "on-chip operand reuse, so `bound` comes from ncu's binding unit"}
    tot = sum(msa[idx[k]] for k in ("fwd_band", "fwd_reduce", "gather_step", "fgp_call",
                                     "snapshot", "other"))
    rec["share_of_profiled_step"] = round(ms[top] / tot, 4) if tot else None
    sub_name = {"fwd_band": "fwd_band", "gather": "gather_step"}.get(top)
    if sub_name:  # per launch: the subset launches and the snapshot's all-angle launch
        i, j = idx[sub_name], idx["snap_" + ("fwd_band" if top == "fwd_band" else "gather")]
        rec["subset_launch_us"] = round(1e3 * msa[i] / cnt[i], 2) if cnt[i] else None
        rec["snapshot_launch_us"] = round(1e3 * msa[j] / cnt[j], 2) if cnt[j] else None
    b = ncu_binding(cfg.name, kernel)
    if b:
        fr = {"issue": b.get("issue_frac"), "lsu": b.get("lsu_shared_frac"),
              "hbm": b.get("dram_frac")}
        fr = {k: v for k, v in fr.items() if v is not None}
        rec["bound"] = max(fr, key=fr.get) if fr else None
        rec["binding"] = {"issue_frac": b.get("issue_frac"),
                          "lsu_shared_frac": b.get("lsu_shared_frac"),
                          "dram_frac": b.get("dram_frac"), "l2_hit": b.get("l2_hit"),
                          "bank_conflict_share": b.get("bank_conflict_share"),
                          "ncu_us": b.get("us"), "source": b.get("source")}
        # ncu bytes of one launch; per call for the FGP (launches per call)
        per = b.get("dram_bytes")
        if per is not None:
            rec["traffic"] = per * b.get("launches_per_call", 1)
            rec["traffic_unit"] = "bytes per call (ncu dram__bytes_read+write, same config)"
    return rec


# --------------------------------------------------------------------------
# process group: --gpus N spawns N ranks itself
# --------------------------------------------------------------------------

def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(args):
    """`python bench.py --gpus N` without torchrun: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1 rendezvous),
    refusing to run with fewer than N visible GPUs."""
    if not args.dry_run and args.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible", file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world):
    """Form the process group exactly as the GPU arm does (gloo instead of
    NCCL, no device work) and report its size."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.ones(1)
    dist.all_reduce(t)
    if world != args.gpus:
        raise SystemExit(f"process group has {world} ranks, --gpus {args.gpus}")
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": args.gpus, "world": dist.get_world_size(),
                          "allreduce_sum": float(t.item())}), flush=True)
    dist.destroy_process_group()
    return 0


def gpu_arm(args, cfg, rank, world, local):
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dp = world > 1 or args.dp_one_rank  # the multi-GPU data path
    if dp:
        if "RANK" not in os.environ:  # --dp-one-rank without torchrun: a one-rank group
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if world != max(1, args.gpus) and not args.dp_one_rank:
            raise SystemExit(f"NCCL group has {world} ranks, --gpus {args.gpus}")
    from paper_2602_09527_b200 import SolverConfig, TomoProblem, run
    from paper_2602_09527_b200 import _native as N
    from paper_2602_09527_b200 import distributed as D
    from paper_2602_09527_b200.solvers import _init_state, _plan_segment

    proj, b_host, b_dev, problem, gamma, alpha = build_gpu_problem(cfg, torch)
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=1e18, seed=cfg.solver_seed)
    stream = torch.cuda.Stream()
    # multi-GPU: angle sectors or image rows (2D), z-slabs (slice-stacked 3D);
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
        return subs, thetas, refr

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
    subs, thetas, refr = run_epochs(args.steps)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = N.launch_count() - launches0
    clock_info = clocks.stop()
    n_iter, n_prox = len(subs), int(np.count_nonzero(thetas))
    ms = t_start.elapsed_time(t_end)
    if dp:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    bad = sess.bad_iteration()
    value = args.steps / (ms / 1e3)

    # replicas exist only in the angle-sector layout (slab layouts own disjoint parts)
    replicas_ok = D.replicas_identical(sess.x) if (dp and zs is None and rs is None) else None

    # live per-kernel timing: the same number of epochs again (the trajectory
    # continues) with CUDA events around every launch category
    roofline = None
    kernel_times = None
    if not args.no_profile:
        import ctypes
        N.check(N.lib().pt_session_set_profiling(sess.handle, 1))
        psubs, pthetas, prefr = run_epochs(args.steps)
        nc = len(N.PROF_NAMES)
        msa = (ctypes.c_double * nc)()
        cnt = (ctypes.c_int64 * nc)()
        N.check(N.lib().pt_session_profile(sess.handle, msa, cnt))
        N.check(N.lib().pt_session_set_profiling(sess.handle, 0))
        top_level = ("fwd_band", "fwd_reduce", "gather_step", "fgp_call", "snapshot", "other")
        tot = sum(msa[N.PROF_NAMES.index(k)] for k in top_level)
        kernel_times = {name: {"ms": round(msa[i], 3), "calls": int(cnt[i]),
                               "share": round(msa[i] / tot, 4) if tot else None}
                        for i, name in enumerate(N.PROF_NAMES)}
        kernel_times["_note"] = ("top-level categories partition the profiled epochs; snap_* "
                                 "are the snapshot's own launches (inside 'snapshot')")
        wp = work.projector
        depth = getattr(wp, "n_slices", 1)
        n_px = wp.width * wp.height * depth
        own = owned_angles(cfg, rank, world, dp and zs is None and rs is None)
        alg, nnz0, _ = epoch_algorithmic_bytes(cfg, wp.plan, psubs, prefr,
                                               int(np.count_nonzero(pthetas)), n_px, depth, own)
        peak, peak_kind = peaks()
        roofline = roofline_record(cfg, msa, cnt, alg, peak, peak_kind)
        if roofline:
            roofline["nnz_subset0"] = nnz0

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
            "config": bench_config(cfg),
            "step": "1 epoch (snapshot + N iterations) of one continuing trajectory",
            "parallelism": ("1 GPU" if not dp else
                            f"z-slab dp{world}" if zs else
                            f"image-row dp{world}" if rs else
                            f"angle-sector dp{world} (replicated image, "
                            f"{'row-sharded' if sector_prox_sharded(world) else 'replicated'} "
                            f"prox)"),
            "timed": {"epochs": args.steps, "iterations": n_iter, "prox_calls": n_prox,
                      "snapshots": int(np.count_nonzero(refr))},
            "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clock_info, "kernel_times": kernel_times,
            "problem": {"L": POWER_L[cfg.name], "gamma": gamma, "alpha": alpha},
            "finite": bad is None, "replicas_identical": replicas_ok,
            "nccl_ranks": world if dp else None,
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)
    if args.dry_run:
        return dry_run(args, rank, world)
    from paper_2602_09527_b200 import problems
    cfg = problems.CONFIGS[args.config]
    if args.impl == "reference":
        return reference_arm(args, cfg, rank, world)
    return gpu_arm(args, cfg, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
