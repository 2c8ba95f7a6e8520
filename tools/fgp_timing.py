"""FGP-100 timing at 2048^2 (warm GPU: 20 untimed calls, then 10 timed)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import TvProxConfig, problems, tv_prox  # noqa: E402

x = torch.tensor(problems.ellipse_phantom(2048, 60, 0), device="cuda", dtype=torch.float32)
for alpha in (0.02,) + ((1.2e-7, 1e-3) if "--all" in sys.argv else ()):
    cfg = TvProxConfig(alpha=alpha, inner_iterations=100)
    out, st = tv_prox(x, 1.0, cfg)
    for _ in range(20):
        out, st = tv_prox(x, 1.0, cfg, warm=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        out, st = tv_prox(x, 1.0, cfg, warm=st)
    e1.record()
    torch.cuda.synchronize()
    print(f"alpha={alpha:g} fgp100 ms {e0.elapsed_time(e1) / 10:.3f} "
          f"dual max {float((st.p ** 2 + st.q ** 2).max()):.3f}")
