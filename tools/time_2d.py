"""Device timing of the 2D fwd / bwd, fused (f2) vs staged, on C3 / C4 / C5 (CUDA events,
L2 flushed before each call, no profiler).

    python tools/time_2d.py [c3|c4|c5 ...] [--reps R]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox, workloads  # noqa: E402

FLUSH = torch.empty((256 << 20) // 4, device="cuda")


def timed(fn, reps):
    t = []
    for _ in range(reps):
        FLUSH.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t.append(a.elapsed_time(b))
    return float(np.median(t))


def run(name, reps):
    w = {"c3": workloads.c3, "c4": workloads.c4, "c5": workloads.c5}[name]()
    X = torch.as_tensor(w.X, device="cuda")
    G = torch.as_tensor(w.grad, device="cuda")
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    mode = {"scalar": _lib.LAM_SCALAR, "channel": _lib.LAM_PER_CHANNEL, "plane": _lib.LAM_PER_PLANE}[w.lam_mode]
    res = {}
    for fused in (0, 1):
        o = tvprox.make_options(fused2d=fused)
        Y, saved, _ = tvprox.tv2d_fwd(X, lam, w.iters, training=True, opts=o)
        GX, gl = tvprox.tv2d_bwd(G, saved, mode, w.iters, want_lam=True, opts=o)
        for _ in range(2):
            tvprox.tv2d_fwd(X, lam, w.iters, training=True, opts=o)
        f = timed(lambda: tvprox.tv2d_fwd(X, lam, w.iters, training=True, opts=o), reps)
        b = timed(lambda: tvprox.tv2d_bwd(G, saved, mode, w.iters, want_lam=True, opts=o), reps)
        torch.cuda.synchronize()
        res[fused] = (f, b, Y.cpu().numpy(), saved.cpu().numpy(), GX.cpu().numpy(), gl.cpu().numpy())
        print("%s %-6s fwd %.3f ms  bwd %.3f ms" % (name, "fused" if fused else "staged", f, b), flush=True)
    same = [np.array_equal(res[0][i].view(np.uint8), res[1][i].view(np.uint8)) for i in (2, 3, 4, 5)]
    print("%s bitwise fused == staged (Y, saved, grad_X, grad_lam): %s" % (name, same), flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = 10
    if "--reps" in sys.argv:
        reps = int(sys.argv[sys.argv.index("--reps") + 1])
    for n in args or ["c3", "c5"]:
        run(n, reps)
