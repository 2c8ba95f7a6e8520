"""Does a CUDA graph of a whole segment run faster on the device than the
PDL launch chain?  Captures session.run(steps) of config c0/c1 on a side
stream, replays it, and compares device times with the stream-launched run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2602_09527_b200 import SolverConfig, TomoProblem, problems  # noqa: E402
from paper_2602_09527_b200 import solvers as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c0"
cfg = problems.CONFIGS[name]
proj, b_host, b_dev, problem, gamma, alpha = bench.build_gpu_problem(cfg, torch)
ecfg = SolverConfig(gamma=gamma, skip_probability=cfg.p, n_subsets=cfg.n_subsets,
                    estimator=cfg.estimator, max_data_passes=60.0, seed=cfg.solver_seed)
stream = torch.cuda.Stream()
with torch.cuda.stream(stream):
    prob = TomoProblem(proj, b_host, tv=problem.tv)
    st = S._init_state(ecfg, prob, None, stream)
    parts = []
    floor = 0
    while True:
        subs, th, rf, passes, done = S._plan_segment(st, ecfg, floor)
        parts.append((subs, th, rf))
        st.data_passes = passes
        floor = int(np.floor(passes + 1e-12))
        if done:
            break
subs, th, rf = [np.concatenate([p[i] for p in parts]) for i in range(3)]
print(f"{name}: {len(subs)} steps", flush=True)


def timed(fn, reps=5):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), float(np.median(out))


print("stream  min/median ms: %.3f / %.3f" % timed(lambda: st.session.run(subs, th, rf, 0)), flush=True)
g = torch.cuda.CUDAGraph()


def replay():
    with torch.cuda.stream(stream):
        g.replay()



torch.cuda.synchronize()
try:
    with torch.cuda.graph(g, stream=stream):
        st.session.run(subs, th, rf, 0)
    print("graph   min/median ms: %.3f / %.3f" % timed(replay), flush=True)
except Exception as exc:  # noqa: BLE001
    print("capture failed:", exc)
