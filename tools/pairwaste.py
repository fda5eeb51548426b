"""Waste of lockstep line pairs: mean over warps of max(iterations of the lines a warp holds)
vs the mean per line, for C5's cold row pass (1D view of the rows) and C3's rows."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import tvprox, workloads  # noqa: E402

for name, G in (("c5", 2), ("c3", 4), ("c4", 1)):
    w = getattr(workloads, name)()
    X = torch.as_tensor(w.X, device="cuda")
    N, C, H, W = X.shape
    rows = X.reshape(N * C * H, W)
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(
        np.repeat(np.tile(w.lam.astype(np.float32), N), H), device="cuda")
    x, m, it = tvprox.tv1d_fwd(rows, lam, want_iters=True)
    itn = (it.cpu().numpy() & 0xffff).astype(np.float64)
    per_line = itn.mean()
    if G > 1:
        warp = itn[: len(itn) // G * G].reshape(-1, G).max(1).mean()
    else:
        warp = per_line
    # 2 warps per... rows are lines; G lines per warp
    print("%s cold rows: mean per line %.2f, mean of max over %d-line warps %.2f (waste %.1f%%)" % (
        name, per_line, G, warp, 100 * (warp / per_line - 1)), flush=True)
