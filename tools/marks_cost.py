"""What the per-row events of run()'s one-call path cost on the device.

Runs the same planned trajectory three ways on a fresh session each time:
events at every log row (run()'s path), one event at the end, and a plain
pt_session_run (no marks).  Prints device milliseconds per variant.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_09527_b200 import SolverConfig, TomoProblem, problems  # noqa: E402
from paper_2602_09527_b200 import solvers as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = problems.CONFIGS[name]
proj, b_host, b_dev, problem, gamma, alpha = bench.build_gpu_problem(cfg, torch)
ecfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                    estimator=cfg.estimator, max_data_passes=float(epochs), seed=cfg.solver_seed)
stream = torch.cuda.current_stream()


def plan(st):
    parts, marks, n = [], [], 0
    floor = 0
    while True:
        subs, th, rf, passes, done = S._plan_segment(st, ecfg, floor)
        parts.append((subs, th, rf))
        n += len(subs)
        marks.append(n)
        st.data_passes = passes
        floor = int(np.floor(passes + 1e-12))
        if done:
            return [np.concatenate([p[i] for p in parts]) for i in range(3)], marks


def once(mode):
    prob = TomoProblem(proj, b_host, tv=problem.tv)
    st = S._init_state(ecfg, prob, None, stream)
    (subs, th, rf), marks = plan(st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    if mode == "rows":
        evs = [torch.cuda.Event(enable_timing=True) for _ in marks]
        for e in evs:
            e.record(stream)
        e0.record(stream)
        st.session.run_marked(subs, th, rf, 0, marks, evs)
    elif mode == "end":
        e1.record(stream)  # materialise the handle
        e0.record(stream)
        st.session.run_marked(subs, th, rf, 0, [marks[-1]], [e1])
    else:
        st.session.run(subs, th, rf, 0)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), len(marks), len(subs)


for rep in range(3):
    for mode in ("rows", "end", "plain"):
        ms, nm, ns = once(mode)
        print(f"{name} rep {rep} {mode:5s}: {ms:.3f} ms  ({nm} marks, {ns} steps)", flush=True)
