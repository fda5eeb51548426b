"""Degenerate-tie stress (integer rows, half-integer lambda) for one library build:
non-converged rows, stall accepts and the max error against the oracle per (n, dtype).

    python tools/ab_lib.py <lib.so> tools/degen_check.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2204_03643_b200 import tvprox, workloads  # noqa: E402

for dt, npdt in (("f32", np.float32), ("f64", np.float64)):
    for n in (17, 56, 100, 224, 300, 512, 1024, 3000):
        y = workloads.random_rows(7400 + n, 64, n, "int", npdt)
        lam = np.random.default_rng(n + 1).integers(1, 7, 64) * 0.5
        x, m, it = tvprox.tv1d_fwd(torch.as_tensor(y, device="cuda"), torch.as_tensor(lam.astype(npdt), device="cuda"),
                                   want_iters=True)
        it = it.cpu().numpy()
        xr, _, _ = oracle.prox1d_batch(y.astype(np.float64), lam, nthreads=8)
        err = np.abs(x.cpu().numpy().astype(np.float64) - xr).max() / max(np.ptp(y), 1e-30)
        print("%s n %5d  not converged %2d  stall-accepted %2d  iters max %3d  max err/range %.2e" % (
            dt, n, (it < 0).sum(), ((it >= 0) & ((it >> 16) & 1 == 1)).sum(), (it[it >= 0] & 0xffff).max(), err),
            flush=True)
