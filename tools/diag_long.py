"""Convergence diagnostics of long 1D rows (f4): PN iteration histogram per option set."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import tvprox  # noqa: E402


DT = np.float64 if os.environ.get("DIAG_F64") else np.float32


def rows(n, nr, seed=0):
    rng = np.random.default_rng(seed)
    y = np.zeros((nr, n), np.float32)
    y[:, n // 2:] = 1.0
    y += (rng.standard_normal((nr, n)) * np.where(np.arange(nr) % 2 == 0, 0.1, 0.5)[:, None]).astype(np.float32)
    lam = rng.uniform(0.13, 1.3, nr).astype(np.float32) * np.float32(np.sqrt(n / 1024))
    return torch.as_tensor(y.astype(DT), device="cuda"), torch.as_tensor(lam.astype(DT), device="cuda")


for n in [int(v) for v in sys.argv[1:]] or [4096, 8192, 16384]:
    y, lam = rows(n, 256)
    for ls_after in (0,):
        for fl in ("backtrack",):
            diag = torch.zeros(4, dtype=torch.int32, device="cuda")
            o = tvprox.make_options(line_search=fl, ls_after=ls_after, diag=diag)
            x, m, it = tvprox.tv1d_fwd(y, lam, want_iters=True, opts=o)
            itn = it.cpu().numpy()
            nc = (itn < 0).sum()
            c = (itn[itn >= 0] & 0xffff)
            st = ((itn[itn >= 0] >> 16) & 1).sum()
            print("n %6d ls_after %2d %-9s not conv %3d / %d  iters mean %.1f p50 %d p90 %d max %d  stall %d  ls rows %d passes %d" % (
                n, ls_after, fl, nc, len(itn), c.mean(), np.percentile(c, 50), np.percentile(c, 90), c.max(), st,
                diag[1].item(), diag[2].item()), flush=True)
