"""The differentiable TV layer of Sec. 3.1 (Eq. 3-4, Fig. 2), NEXT row f1.

    layer = TVLayer(num_chan=C, is_sharp=False, mode="2d", iters=4)
    Y = layer(X)          # X [N, C, H, W] CUDA fp32/fp64

lambda_c = SoftPlus(lambda-tilde_c).  lambda-tilde is initialised so that lambda = 0.05,
the paper's initialisation for the TV layers it inserts into networks (Sec. 4.2, P:313:
"initialize lambda = 0.05"); init=0.0 gives Fig. 2's zero-initialised lambda-tilde
(lambda = ln 2).  Smoothing Y_c = Prox(X_c, lambda_c) (Eq. 3) or sharpening
Y_c = 2 X_c - Prox(X_c, lambda_c) (Eq. 4); spatial mode "2d" (anisotropic 2D prox by
K Proximal-Dykstra iterations, Alg. 1), "rows" or "cols" (a 1D prox per row or per
column).  Every step (SoftPlus, prox, sharpen, and their VJPs) runs in
libtvprox.so kernels; torch supplies parameters, memory and the stream.
"""
from __future__ import annotations

import math

import torch

from . import _lib, tvprox


class _SoftPlus(torch.autograd.Function):
    @staticmethod
    def forward(ctx, t):
        ctx.save_for_backward(t)
        return tvprox.softplus_fwd(t)

    @staticmethod
    def backward(ctx, g):
        (t,) = ctx.saved_tensors
        return tvprox.softplus_bwd(t, g)


class _Sharpen(torch.autograd.Function):
    """Y = 2 X - P  with P = prox(X) computed upstream; VJP: dX = 2 G, dP = -G."""

    @staticmethod
    def forward(ctx, X, P):
        Y = P.contiguous().clone()
        return tvprox.axpby_(X.contiguous(), Y, 2.0, -1.0)

    @staticmethod
    def backward(ctx, G):
        G = G.contiguous()
        gX = tvprox.axpby_(G, torch.empty_like(G), 2.0, 0.0)
        gP = tvprox.axpby_(G, torch.empty_like(G), -1.0, 0.0)
        return gX, gP


def tv_layer(X: torch.Tensor, lam_tilde: torch.Tensor, is_sharp: bool = False, mode: str = "2d",
             iters: int = 4) -> torch.Tensor:
    lam = _SoftPlus.apply(lam_tilde)
    if mode == "2d":
        P = tvprox.tv2d(X, lam, iters=iters)
    elif mode == "rows":
        P = tvprox.tv2d_lines(X, lam, 0)
    elif mode == "cols":
        P = tvprox.tv2d_lines(X, lam, 1)
    else:
        raise ValueError("mode must be '2d', 'rows' or 'cols'")
    return _Sharpen.apply(X, P) if is_sharp else P


LAM_INIT = 0.05
INIT_LAM_TILDE = float(math.log(math.expm1(LAM_INIT)))   # softplus^-1(0.05)


class TVLayer(torch.nn.Module):
    """shared=True: one lambda-tilde for all channels ("lambda shared across channels",
    P:313); the kernels still see a per-channel lambda (the expanded value), so the
    call stays asynchronous and the gradient is the sum over channels."""

    def __init__(self, num_chan: int, is_sharp: bool = False, mode: str = "2d", iters: int = 4,
                 init: float = INIT_LAM_TILDE, dtype=torch.float32, device=None, shared: bool = False):
        super().__init__()
        self.is_sharp = is_sharp
        self.mode = mode
        self.iters = iters
        self.num_chan = num_chan
        self.shared = shared
        self._lmbd = torch.nn.Parameter(torch.full((1 if shared else num_chan,), float(init), dtype=dtype,
                                                   device=device))

    def _lam_tilde(self) -> torch.Tensor:
        return self._lmbd.expand(self.num_chan) if self.shared else self._lmbd

    @property
    def lam(self) -> torch.Tensor:
        return tvprox.softplus_fwd(self._lam_tilde().detach().contiguous())

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return tv_layer(x, self._lam_tilde(), self.is_sharp, self.mode, self.iters)
