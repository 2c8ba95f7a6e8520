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
