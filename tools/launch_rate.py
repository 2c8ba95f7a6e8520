"""Host enqueue time vs device time of a native segment (launch-bound
configs): c0 / c1 sessions, `steps` ProxSkip iterations in one
pt_session_run call."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_09527_b200 import SolverConfig, problems  # noqa: E402
from paper_2602_09527_b200.solvers import _init_state, _plan_segment  # noqa: E402

for name in sys.argv[1:] or ["c0", "c1"]:
    cfg = problems.CONFIGS[name]
    proj, b_host, b_dev, problem, gamma, alpha = bench.build_gpu_problem(cfg, torch)
    scfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                        estimator=cfg.estimator, max_data_passes=1e18, seed=cfg.solver_seed)
    st = _init_state(scfg, problem, None)
    for rep in range(4):
        subs, th, rf, passes, _ = _plan_segment(st, scfg, 1 << 62, max_steps=20 * cfg.n_subsets)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        st.session.run(subs, th, rf, st.k)
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st.k += len(subs)
        n = len(subs)
        print(f"{name} rep {rep}: {n} steps, host enqueue {1e6 * (t1 - t0) / n:.1f} us/step, "
              f"device {1e3 * e0.elapsed_time(e1) / n:.1f} us/step, wall {1e6 * (t2 - t0) / n:.1f} "
              f"us/step, prox {int(np.count_nonzero(th))}", flush=True)
