"""Small-shape invocation of every kernel (for compute-sanitizer memcheck/racecheck/synccheck/initcheck).

    compute-sanitizer --tool memcheck python tools/sanitize.py [quick]

Covers: 1D rows of every register geometry (staged, register-direct, two-warp, one-CTA long
rows and thread-block-cluster rows past 8192 samples), scalar / per-row / per-edge lambda,
warm starts, both line-search flavours; 2D staged passes, the fused 56^2 plane kernel and
the thread-block-cluster planes (fused2d = 1), inference and training; the TV-layer helpers.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox  # noqa: E402

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
rng = np.random.default_rng(0)
for dt in (torch.float32, torch.float64):
    ns = (1, 2, 17, 33, 56, 64, 100, 224, 300, 512, 700, 1024, 2000, 5000)
    if not quick:
        ns = ns + ((9000, 20000) if dt == torch.float32 else (4500, 9000))
    for n in ns:
        b = 5 if n <= 5000 else 2
        y = torch.as_tensor(rng.standard_normal((b, n)), dtype=dt, device="cuda")
        for lam in (0.4, torch.full((b,), 0.3, dtype=dt, device="cuda"),
                    torch.full((b, max(n - 1, 1)), 0.2, dtype=dt, device="cuda")):
            x, m, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
            mode = _lib.LAM_SCALAR if not torch.is_tensor(lam) else (_lib.LAM_PER_ROW if lam.dim() == 1 else _lib.LAM_PER_EDGE)
            tvprox.tv1d_bwd(y, m, mode)
            tvprox.tv1d_fwd(y, lam, warm_mask=m)
        for fl in ("backtrack", "parallel"):
            tvprox.tv1d_fwd(y, 0.7, opts=tvprox.make_options(line_search=fl, ls_after=2))
    shapes = ((1, 5), (7, 1), (3, 4), (56, 56), (40, 61), (33, 224), (224, 33), (130, 520))
    for (H, W) in shapes:
        X = torch.as_tensor(rng.standard_normal((2, 2, H, W)), dtype=dt, device="cuda")
        lam = torch.tensor([0.3, 0.8], dtype=dt, device="cuda")
        for fused in (0, 1):
            o = tvprox.make_options(fused2d=fused)
            Y, saved, it = tvprox.tv2d_fwd(X, lam, 3, want_iters=True, opts=o)
            tvprox.tv2d_bwd(X, saved, _lib.LAM_PER_CHANNEL, 3, opts=o)
            tvprox.tv2d_fwd(X, 0.5, 2, training=False, opts=o)
        tvprox.tv2d_fwd(X, lam, 2, opts=tvprox.make_options(line_search="parallel", ls_after=2))
    if dt == torch.float32:
        # thread-block-cluster planes (f2, fused2d = 1): both geometries, ragged partitions
        for (H, W) in ((224, 224), (150, 200), (97, 65)):
            X = torch.as_tensor(rng.standard_normal((1, 2, H, W)), dtype=dt, device="cuda")
            o = tvprox.make_options(fused2d=1)
            Y, saved, _ = tvprox.tv2d_fwd(X, torch.tensor([0.3, 0.8], device="cuda"), 3, opts=o)
            tvprox.tv2d_bwd(X, saved, _lib.LAM_PER_CHANNEL, 3, opts=o)
            tvprox.tv2d_fwd(X, 0.5, 2, training=False, opts=o)
        # TV layer helpers (f1)
        t = torch.randn(8, device="cuda")
        lamv = tvprox.softplus_fwd(t)
        X = torch.randn(2, 3, 20, 30, device="cuda")
        for axis in (0, 1):
            Yl, ml = tvprox.tv2d_lines_fwd(X, torch.tensor([0.2, 0.5, 0.9], device="cuda"), axis)
            tvprox.tv2d_lines_bwd(X, ml, _lib.LAM_PER_CHANNEL, axis)
torch.cuda.synchronize()
print("sanitize workload done")
