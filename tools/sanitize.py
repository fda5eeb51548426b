"""Small-shape invocation of every kernel (for compute-sanitizer memcheck/racecheck/synccheck/initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox  # noqa: E402

rng = np.random.default_rng(0)
for dt in (torch.float32, torch.float64):
    for n in (1, 2, 17, 33, 56, 64, 100, 224, 300, 512, 700, 1024):
        y = torch.as_tensor(rng.standard_normal((5, n)), dtype=dt, device="cuda")
        for lam in (0.4, torch.full((5,), 0.3, dtype=dt, device="cuda"),
                    torch.full((5, max(n - 1, 1)), 0.2, dtype=dt, device="cuda")):
            x, m, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
            mode = _lib.LAM_SCALAR if not torch.is_tensor(lam) else (_lib.LAM_PER_ROW if lam.dim() == 1 else _lib.LAM_PER_EDGE)
            tvprox.tv1d_bwd(y, m, mode)
            tvprox.tv1d_fwd(y, lam, warm_mask=m)
    for (H, W) in ((1, 5), (7, 1), (3, 4), (56, 56), (33, 224), (224, 33), (130, 520)):
        X = torch.as_tensor(rng.standard_normal((2, 2, H, W)), dtype=dt, device="cuda")
        lam = torch.tensor([0.3, 0.8], dtype=dt, device="cuda")
        Y, saved, it = tvprox.tv2d_fwd(X, lam, 3, want_iters=True)
        tvprox.tv2d_bwd(X, saved, _lib.LAM_PER_CHANNEL, 3)
        tvprox.tv2d_fwd(X, 0.5, 2, training=False)
torch.cuda.synchronize()
print("sanitize workload done")
