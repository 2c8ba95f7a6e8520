"""Host-side breakdown of run() at a small configuration (where e2e < value)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_09527_b200 import SolverConfig, TomoProblem, problems, run  # noqa: E402
from paper_2602_09527_b200 import solvers as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
cfg = problems.CONFIGS[name]
proj, b_host, b_dev, problem, gamma, alpha = bench.build_gpu_problem(cfg, torch)
ecfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                    estimator=cfg.estimator, max_data_passes=3.0 * 20, seed=cfg.solver_seed)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = TomoProblem(proj, b_host, tv=problem.tv)
    t1 = time.perf_counter()
    st = S._init_state(ecfg, prob, None, torch.cuda.current_stream())
    t2 = time.perf_counter()
    rec = S._run_loop(st, ecfg, prob, None, None, False, torch.cuda.current_stream())
    t3 = time.perf_counter()
    img = rec.image.cpu()
    t4 = time.perf_counter()
    print(f"rep {rep}: problem {1e3*(t1-t0):.2f} ms  init_state {1e3*(t2-t1):.2f} ms  "
          f"run_loop {1e3*(t3-t2):.2f} ms  d2h {1e3*(t4-t3):.2f} ms  device work "
          f"{rec.rows[-1][1]*1e3:.2f} ms  rows {len(rec.rows)}", flush=True)
import cProfile, pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
rec = run(ecfg, TomoProblem(proj, b_host, tv=problem.tv))
rec.image.cpu()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
