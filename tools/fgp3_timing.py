"""3D FGP-100 timing at 256^3 (config 3's prox), warm duals."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_09527_b200 import TvProxConfig, problems, tv_prox  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
x = torch.tensor(problems.ellipsoid_phantom(n, 40, 0), device="cuda", dtype=torch.float32)
cfg = TvProxConfig(alpha=0.01, inner_iterations=100)
out, st = tv_prox(x, 1.0, cfg)
for _ in range(8):  # warm the GPU clocks
    out, st = tv_prox(x, 1.0, cfg, warm=st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    out, st = tv_prox(x, 1.0, cfg, warm=st)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
vox = n ** 3
print(f"zchunk={os.environ.get('PT_FGP3_ZCHUNK', 'auto')} fgp3d-100 {n}^3 ms {ms:.3f} "
      f"per-iter us {ms * 10:.1f} GB/s(40B/vox) {40 * vox * 100 / ms / 1e6:.0f}")
