"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method: it only draws numbers.  It is
the one module shared by the CUDA path's callers (tests, bench) and the oracle's
callers; neither the oracle nor the CUDA library imports it.

Recipe:
  seeds       1000*config + {0: input, 1: lambda-tilde, 2: upstream gradient}
  C1 (BJ:7)   1D fp64, 8 x 64, lam 0.5; rows 0-3 unit step at 32 + N(0, 0.1^2)
              (Table 1 family), rows 4-7 iid N(0,1)
  C2 (BJ:8)   1D fp32, 65536 x 1024, per-row lam = softplus(U(-2,1));
              unit step at 512 + N(0, sigma_b^2), sigma 0.1 (even b) / 0.5 (odd b);
              seeded per block of 1024 rows ([seed, block]) so row shards are slices
  C3 (BJ:9)   2D fp32 NCHW 64x64x56x56, K=4, per-channel lam =
              softplus(linspace(-3, 0, 64)); X = max(N(0,1), 0) (post-ReLU features)
  C4 (BJ:10)  2D fp32 16x3x512x512, K=4, scalar lam = 1; per plane a background
              level plus 16 axis-aligned rectangles with U(0,1) levels, plus
              N(0, (25/255)^2) noise (sigma = 25)
  C5 (BJ:11)  2D fp32 256x3x224x224, K=4, per-channel lam = softplus((-1,0,1));
              C4's generator at 224^2, then ImageNet normalisation
  T1a/T1b     1D fp32 8192 x 32 and 256 x 1024, lam 1, unit step + N(0, 0.1^2)
              (the two readings of Table 1's "256 x 32 x 32", O17)
Upstream gradients are N(0,1) in the config dtype.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def softplus_np(t):
    """log(1 + e^t): only used to draw positive lambdas the way the layer would."""
    t = np.asarray(t, np.float64)
    return np.log1p(np.exp(-np.abs(t))) + np.maximum(t, 0.0)


@dataclass
class Workload1D:
    name: str
    y: np.ndarray            # [batch, n], config dtype
    lam: np.ndarray          # per-row [batch] or per-edge [batch, n-1] (fp64 values)
    lam_mode: str            # "scalar" | "row" | "edge"
    lam_scalar: float
    dtype: str
    seed: int
    grad: np.ndarray = field(default=None)


@dataclass
class Workload2D:
    name: str
    X: np.ndarray            # [N, C, H, W], config dtype
    lam: np.ndarray          # [C] (per channel) or [N*C] (per plane) or [1]
    lam_mode: str            # "scalar" | "channel" | "plane"
    lam_scalar: float
    iters: int
    dtype: str
    seed: int
    grad: np.ndarray = field(default=None)


def _unit_step(rng, b, n, p, sigma):
    y = np.zeros((b, n))
    y[:, p:] = 1.0
    return y + rng.standard_normal((b, n)) * np.asarray(sigma).reshape(-1, 1)


def rect_planes(rng, planes, H, W, nrect=16, sigma=25.0 / 255.0):
    """Piecewise-constant random rectangles per plane plus Gaussian noise (C4/C5 recipe)."""
    out = np.empty((planes, H, W))
    for p in range(planes):
        img = np.full((H, W), rng.uniform(0.0, 1.0))
        for _ in range(nrect):
            h0, h1 = np.sort(rng.integers(0, H + 1, size=2))
            w0, w1 = np.sort(rng.integers(0, W + 1, size=2))
            if h1 == h0:
                h1 = min(H, h0 + 1)
            if w1 == w0:
                w1 = min(W, w0 + 1)
            img[h0:h1, w0:w1] = rng.uniform(0.0, 1.0)
        out[p] = img
    out += rng.standard_normal(out.shape) * sigma
    return out


def c1(with_grad=True) -> Workload1D:
    seed = 1000 * 1
    rng = np.random.default_rng(seed + 0)
    y = np.empty((8, 64))
    y[:4] = _unit_step(rng, 4, 64, 32, 0.1)
    y[4:] = rng.standard_normal((4, 64))
    g = np.random.default_rng(seed + 2).standard_normal((8, 64)) if with_grad else None
    return Workload1D("C1", y.astype(np.float64), np.full(8, 0.5), "scalar", 0.5, "f64", seed, g)


C2_BLOCK = 1024       # rows per seeding block of C2 (so any row shard is reproducible)


def c2(batch=65536, n=1024, with_grad=True, dtype=np.float32, row_offset=0) -> Workload1D:
    """Rows [row_offset, row_offset + batch) of the C2 family.  Row block j (C2_BLOCK rows)
    draws from its own streams [seed + {0,1,2}, j], so a rank's shard of a multi-GPU batch
    equals the same rows of the single-GPU batch (the N-GPU verification compares them)."""
    seed = 1000 * 2
    b0, b1 = row_offset // C2_BLOCK, (row_offset + batch + C2_BLOCK - 1) // C2_BLOCK
    ys, lts, gs = [], [], []
    for j in range(b0, b1):
        rows = np.arange(j * C2_BLOCK, (j + 1) * C2_BLOCK)
        sig = np.where(rows % 2 == 0, 0.1, 0.5)
        ys.append(_unit_step(np.random.default_rng([seed + 0, j]), C2_BLOCK, n, n // 2, sig).astype(dtype))
        lts.append(np.random.default_rng([seed + 1, j]).uniform(-2.0, 1.0, size=C2_BLOCK))
        if with_grad:
            gs.append(np.random.default_rng([seed + 2, j]).standard_normal((C2_BLOCK, n)).astype(dtype))
    lo = row_offset - b0 * C2_BLOCK
    y = np.ascontiguousarray(np.concatenate(ys)[lo:lo + batch])
    lam = softplus_np(np.concatenate(lts)[lo:lo + batch]).astype(dtype).astype(np.float64)
    g = np.ascontiguousarray(np.concatenate(gs)[lo:lo + batch]) if with_grad else None
    return Workload1D("C2", y, lam, "row", 0.0, "f32", seed, g)


def t1(reading="a", with_grad=True) -> Workload1D:
    b, n = (8192, 32) if reading == "a" else (256, 1024)
    seed = 1000 * 6 + (0 if reading == "a" else 10)
    rng = np.random.default_rng(seed)
    y = _unit_step(rng, b, n, n // 2, 0.1).astype(np.float32)
    g = (np.random.default_rng(seed + 2).standard_normal((b, n)).astype(np.float32)
         if with_grad else None)
    return Workload1D("T1" + reading, y, np.ones(b), "scalar", 1.0, "f32", seed, g)


def long_rows(n, batch=None, with_grad=True) -> Workload1D:
    """f4 ("long 1D signals", BJ:5): C2's generator at length n -- unit step at n/2 plus
    N(0, sigma^2), sigma 0.1 / 0.5 alternating -- with per-row lambda softplus(U(-2, 1))
    scaled by sqrt(n / 1024) (the noise TV grows with sqrt(n)); 2^26 samples per batch."""
    b = batch or max(1, (1 << 26) // n)
    seed = 1000 * 7 + n
    rng = np.random.default_rng(seed)
    y = np.zeros((b, n))
    y[:, n // 2:] = 1.0
    y += rng.standard_normal((b, n)) * np.where(np.arange(b) % 2 == 0, 0.1, 0.5)[:, None]
    lam = softplus_np(np.random.default_rng(seed + 1).uniform(-2.0, 1.0, b)) * np.sqrt(n / 1024.0)
    g = np.random.default_rng(seed + 2).standard_normal((b, n)).astype(np.float32) if with_grad else None
    return Workload1D("L%d" % n, y.astype(np.float32), lam, "row", 0.0, "f32", seed, g)


def c3(N=64, C=64, H=56, W=56, with_grad=True) -> Workload2D:
    seed = 1000 * 3
    rng = np.random.default_rng(seed + 0)
    X = np.maximum(rng.standard_normal((N, C, H, W), dtype=np.float32), 0.0)
    lam = softplus_np(np.linspace(-3.0, 0.0, C)).astype(np.float32).astype(np.float64)
    g = (np.random.default_rng(seed + 2).standard_normal((N, C, H, W), dtype=np.float32)
         if with_grad else None)
    return Workload2D("C3", X, lam, "channel", 0.0, 4, "f32", seed, g)


def c4(N=16, C=3, H=512, W=512, lam=1.0, with_grad=True) -> Workload2D:
    seed = 1000 * 4
    rng = np.random.default_rng(seed + 0)
    X = rect_planes(rng, N * C, H, W).reshape(N, C, H, W).astype(np.float32)
    g = (np.random.default_rng(seed + 2).standard_normal((N, C, H, W), dtype=np.float32)
         if with_grad else None)
    return Workload2D("C4", X, np.array([lam]), "scalar", float(lam), 4, "f32", seed, g)


def c5(N=256, C=3, H=224, W=224, with_grad=True, image_offset=0) -> Workload2D:
    """image_offset selects images [image_offset, image_offset + N) of the full 256-image
    batch deterministically (per-image seeding), so a rank's shard equals the slice."""
    seed = 1000 * 5
    planes = []
    for i in range(image_offset, image_offset + N):
        rng = np.random.default_rng([seed, i])
        planes.append(rect_planes(rng, C, H, W))
    X = np.stack(planes).reshape(N, C, H, W)
    mean = np.array([0.485, 0.456, 0.406]).reshape(1, 3, 1, 1)
    std = np.array([0.229, 0.224, 0.225]).reshape(1, 3, 1, 1)
    X = ((X - mean[:, :C]) / std[:, :C]).astype(np.float32)
    lam = softplus_np(np.array([-1.0, 0.0, 1.0])[:C]).astype(np.float32).astype(np.float64)
    g = None
    if with_grad:
        g = np.stack([np.random.default_rng([seed + 2, i]).standard_normal((C, H, W), dtype=np.float32)
                      for i in range(image_offset, image_offset + N)])
    return Workload2D("C5", X, lam, "channel", 0.0, 4, "f32", seed, g)


def random_rows(seed, batch, n, kind="normal", dtype=np.float64):
    """Generic seeded rows for parity edge cases."""
    rng = np.random.default_rng(seed)
    if kind == "normal":
        y = rng.standard_normal((batch, n))
    elif kind == "step":
        y = _unit_step(rng, batch, n, max(n // 2, 0), 0.1)
    elif kind == "int":
        y = rng.integers(-3, 4, size=(batch, n)).astype(np.float64)
    elif kind == "const":
        y = np.repeat(rng.standard_normal((batch, 1)), n, axis=1)
    else:
        raise ValueError(kind)
    return y.astype(dtype)


CONFIGS = {
    "C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5,
}


def bytes_per_row_1d(n, itemsize=4):
    """Algorithmic bytes of a 1D fwd (or bwd) per row: read n, write n, write the 2-bit mask."""
    return 2 * n * itemsize + 4 * math.ceil(max(n - 1, 0) / 16)
