"""Quick device timing of the hot-path calls (CUDA events, warm, no profiler).

    python tools/time_kernels.py [c2|c3|c4|c5|all]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_03643_b200 import _lib, tvprox, workloads  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def c2():
    w = workloads.c2()
    y = torch.as_tensor(w.y, device="cuda")
    lam = torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    g = torch.as_tensor(w.grad, device="cuda")
    x, mask, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
    itn = it.cpu().numpy()
    f = timeit(lambda: tvprox.tv1d_fwd(y, lam))
    bw = timeit(lambda: tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW))
    gbs = 65536 * (8192 + 260) / 1e9
    print("C2 fwd %.3f ms (%.0f GB/s)  bwd %.3f ms (%.0f GB/s)  iters mean %.2f p99 %d max %d nc %d stall %d" % (
        f, gbs / f * 1e3, bw, gbs / bw * 1e3, (itn & 0xffff).mean(), np.percentile(itn & 0xffff, 99),
        (itn & 0xffff).max(), (itn < 0).sum(), ((itn > 0) & ((itn >> 16) & 1 == 1)).sum()), flush=True)
    # stress: iid normal rows
    ys = torch.randn(65536, 1024, device="cuda")
    x, mask, it = tvprox.tv1d_fwd(ys, 1.0, want_iters=True)
    itn = it.cpu().numpy()
    f = timeit(lambda: tvprox.tv1d_fwd(ys, 1.0))
    print("C2-stress(iid N(0,1), lam 1) fwd %.3f ms iters mean %.2f max %d" % (f, (itn & 0xffff).mean(), (itn & 0xffff).max()), flush=True)


def sweep():
    """ns per (sample x PN iteration) of the 1D forward for each register geometry."""
    rng = np.random.default_rng(0)
    for n in (32, 56, 64, 128, 224, 256, 512, 1024):
        rows = (1 << 26) // n
        y = np.zeros((rows, n), np.float32)
        y[:, n // 2:] = 1.0
        y += (rng.standard_normal((rows, n)) * np.where(np.arange(rows) % 2 == 0, 0.1, 0.5)[:, None]).astype(np.float32)
        yt = torch.as_tensor(y, device="cuda")
        lam = torch.full((rows,), 0.7 * n / 1024 + 0.05, device="cuda")
        x, mask, it = tvprox.tv1d_fwd(yt, lam, want_iters=True)
        itn = (it.cpu().numpy() & 0xffff).astype(np.float64)
        f = timeit(lambda: tvprox.tv1d_fwd(yt, lam), reps=5)
        print("n %5d rows %7d fwd %.3f ms  iters mean %.2f max %d  -> %.3f ns/(sample*iter)  %.1f Gsample/s" % (
            n, rows, f, itn.mean(), itn.max(), f * 1e6 / (rows * n * itn.mean()), rows * n / f / 1e6), flush=True)


def long_rows():
    """f4: long 1D signals (unit step + N(0, 0.1^2) / N(0, 0.5^2) like C2, lambda scaled with n)."""
    rng = np.random.default_rng(0)
    ns = (2048, 4096, 8192, 16384, 32768, 65536) if len(sys.argv) < 3 else tuple(int(v) for v in sys.argv[2:])
    for n in ns:
        rows = (1 << 26) // n
        y = np.zeros((rows, n), np.float32)
        y[:, n // 2:] = 1.0
        y += (rng.standard_normal((rows, n)) * np.where(np.arange(rows) % 2 == 0, 0.1, 0.5)[:, None]).astype(np.float32)
        yt = torch.as_tensor(y, device="cuda")
        lam = torch.as_tensor(rng.uniform(0.13, 1.3, rows).astype(np.float32) * np.float32(np.sqrt(n / 1024)),
                              device="cuda")
        x, mask, it = tvprox.tv1d_fwd(yt, lam, want_iters=True)
        itn = (it.cpu().numpy() & 0xffff)
        f = timeit(lambda: tvprox.tv1d_fwd(yt, lam), reps=5)
        g = torch.randn_like(yt)
        bw = timeit(lambda: tvprox.tv1d_bwd(g, mask, _lib.LAM_PER_ROW), reps=5)
        print("long n %5d rows %6d fwd %.3f ms bwd %.3f ms -> %.1f M rows/s fwd+bwd, %.2f Gsample/s; iters mean %.2f max %d" % (
            n, rows, f, bw, rows / (f + bw) / 1e3, rows * n / (f + bw) / 1e6, itn.mean(), itn.max()), flush=True)


def twod(name):
    w = getattr(workloads, name)()
    X = torch.as_tensor(w.X, device="cuda")
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    G = torch.as_tensor(w.grad, device="cuda")
    mode = {"scalar": 0, "channel": 3, "plane": 4}[w.lam_mode]
    Y, saved, it = tvprox.tv2d_fwd(X, lam, w.iters, want_iters=True)
    f = timeit(lambda: tvprox.tv2d_fwd(X, lam, w.iters), reps=5)
    bw = timeit(lambda: tvprox.tv2d_bwd(G, saved, mode, w.iters), reps=5)
    px = X.numel()
    print("%s fwd %.3f ms bwd %.3f ms  -> %.0f Mpx/s fwd+bwd; max iters/pass %s" % (
        name.upper(), f, bw, px / ((f + bw) * 1e-3) / 1e6, it.cpu().numpy().tolist()), flush=True)


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    if which in ("sweep",):
        sweep()
    if which in ("c2", "all"):
        c2()
    if which in ("long",):
        long_rows()
    for n in ("c3", "c4", "c5"):
        if which in (n, "all"):
            twod(n)
