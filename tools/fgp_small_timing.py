"""2D FGP-100 timing at a given size (default 512^2, config 1's prox)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import TvProxConfig, problems, tv_prox  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = torch.tensor(problems.ellipse_phantom(n, 30, 0), device="cuda", dtype=torch.float32)
cfg = TvProxConfig(alpha=0.02, inner_iterations=100)
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
print(f"n={n} T={os.environ.get('PT_FGP_T', '8')} big_min={os.environ.get('PT_FGP_BIG_MIN', '256')} "
      f"fgp100 us {e0.elapsed_time(e1) * 100:.1f}")
