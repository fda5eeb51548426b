"""Outputs of one libtvprox build on fixed inputs, for a bitwise comparison of two builds.

    python tools/bitcmp.py <lib.so> <out.npz>; python tools/bitcmp_cmp.py a.npz b.npz
"""
import sys, os
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2204_03643_b200 import _lib
_lib.load(sys.argv[1])
from paper_2204_03643_b200 import tvprox, workloads
out = {}
rng = np.random.default_rng(0)
for n in (20, 56, 100, 128, 200, 224, 512, 777, 1024, 2048, 3001):
    for dt in (torch.float32, torch.float64):
        y = torch.as_tensor(rng.standard_normal((301, n)), dtype=dt, device="cuda")
        lam = torch.as_tensor(rng.uniform(0.1, 2.0, 301), dtype=dt, device="cuda")
        x, m, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
        out["1d_%d_%s" % (n, dt)] = x.cpu().numpy()
        out["1d_it_%d_%s" % (n, dt)] = it.cpu().numpy()
        out["1d_mask_%d_%s" % (n, dt)] = m.cpu().numpy()
        x0, m0, _ = tvprox.tv1d_fwd(y, 0.0, want_iters=True)             # lam = 0: boundary codes
        out["1d_mask0_%d_%s" % (n, dt)] = m0.cpu().numpy()
for H, W in ((56, 56), (224, 224), (100, 37), (129, 300)):
    X = torch.as_tensor(rng.standard_normal((2, 3, H, W)), dtype=torch.float32, device="cuda")
    Y, saved, it = tvprox.tv2d_fwd(X, torch.tensor([0.2, 0.7, 1.5], device="cuda"), 4, want_iters=True)
    out["2d_%d_%d" % (H, W)] = Y.cpu().numpy()
w = workloads.c5(N=8)
X = torch.as_tensor(w.X, device="cuda")
Y, _, _ = tvprox.tv2d_fwd(X, torch.as_tensor(w.lam.astype(np.float32), device="cuda"), 4)
out["c5"] = Y.cpu().numpy()
np.savez(sys.argv[2], **out)
print("saved", len(out))
