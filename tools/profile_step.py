"""Run a few steps of one workload's hot path (for ncu captures under gpurun).

    python tools/profile_step.py c2|c3|c4|c5 [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox, workloads  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda", 0)
    if wl == "c2":
        w = workloads.c2()
        y = torch.as_tensor(w.y, device=dev)
        lam = torch.as_tensor(w.lam.astype(np.float32), device=dev)
        g = torch.as_tensor(w.grad, device=dev)
        for _ in range(steps):
            x, mask, _ = tvprox.tv1d_fwd(y, lam)
            tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW)
    else:
        w = getattr(workloads, wl)()
        X = torch.as_tensor(w.X, device=dev)
        lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device=dev)
        G = torch.as_tensor(w.grad, device=dev)
        mode = {"scalar": 0, "channel": 3, "plane": 4}[w.lam_mode]
        for _ in range(steps):
            Y, saved, _ = tvprox.tv2d_fwd(X, lam, w.iters)
            tvprox.tv2d_bwd(G, saved, mode, w.iters)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
