"""PyTorch binding of libtvprox.so (argument marshalling only).

PyTorch provides device memory and the current CUDA stream; every step of the
TV prox runs in the library's sm_100a kernels.  CPU tensors are rejected: there
is no CPU fallback on the product path.

    x = tv1d(y, lam)                  # y [batch, n] CUDA fp32/fp64; lam float | [batch] | [batch, n-1]
    Y = tv2d(X, lam, iters=4)         # X [N, C, H, W]; lam float | [C] | [N*C] (or [N, C])
Both are autograd-aware (Eq. 7-8 backward for 1D, reverse mode through
Algorithm 1 for 2D).
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import check

_DT = {torch.float32: _lib.TVP_F32, torch.float64: _lib.TVP_F64}


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise TypeError("tvprox: dtype must be float32 or float64, got %s" % t.dtype)
    return _DT[t.dtype]


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("tvprox: tensors must live on a CUDA device (no CPU fallback)")


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def make_options(fused2d: int = -1, line_search: str = "backtrack", ls_after: int = 0, diag: torch.Tensor = None,
                 iter_hist: torch.Tensor = None):
    """tvp_options_t for the *_ex calls (include/tvprox.h).  diag: int32 CUDA [4];
    iter_hist: int32 CUDA [passes, HIST_BINS] (both accumulated by the call)."""
    ls = {"backtrack": _lib.LS_BACKTRACK, "parallel": _lib.LS_PARALLEL}[line_search]
    for t in (diag, iter_hist):
        if t is not None:
            _require_cuda(t)
            if t.dtype != torch.int32 or not t.is_contiguous():
                raise ValueError("tvprox: diag / iter_hist must be contiguous int32")
    return _lib.Options(int(fused2d), ls, int(ls_after), _ptr(diag), _ptr(iter_hist))


def _opts_ref(opts):
    import ctypes
    return None if opts is None else ctypes.byref(opts)


def _rows(y: torch.Tensor) -> torch.Tensor:
    if y.dim() != 2:
        raise ValueError("tvprox: 1D input must be [batch, n]")
    if y.stride(1) != 1 or (y.shape[0] > 1 and y.stride(0) < y.shape[1]):
        y = y.contiguous()
    return y


def _lam1d(lam, y: torch.Tensor):
    """-> (mode, scalar, tensor or None) with per-edge lam laid out with y's row pitch."""
    if not torch.is_tensor(lam):
        return _lib.LAM_SCALAR, float(lam), None
    lam = lam.to(device=y.device, dtype=y.dtype)
    b, n = y.shape
    if lam.dim() == 0:
        return _lib.LAM_SCALAR, float(lam.item()), None
    if lam.dim() == 1:
        if lam.shape[0] != b:
            raise ValueError("tvprox: per-row lam must have shape [batch]")
        return _lib.LAM_PER_ROW, 0.0, lam.contiguous()
    if lam.dim() == 2 and lam.shape[0] == b and lam.shape[1] in (n - 1, n, y.stride(0)):
        pitch = y.stride(0) if b > 1 else n
        if lam.shape[1] != pitch or lam.stride(1) != 1 or (b > 1 and lam.stride(0) != pitch):
            full = torch.zeros((b, pitch), device=y.device, dtype=y.dtype)
            m = min(lam.shape[1], n - 1)
            full[:, :m] = lam[:, :m]
            lam = full
        return _lib.LAM_PER_EDGE, 0.0, lam
    raise ValueError("tvprox: lam must be a float, [batch] or [batch, n-1]")


def tv1d_fwd(y: torch.Tensor, lam, need_mask: bool = True, want_iters: bool = False,
             warm_mask: torch.Tensor = None, opts=None):
    """Batched 1D TV prox forward.  Returns (x, mask or None, row_iters or None).
    warm_mask: optional saved mask of a previous solve to warm-start projected Newton.
    opts: optional make_options(...) (line-search flavour, diagnostics)."""
    _require_cuda(y)
    y = _rows(y)
    dt = _dtype_code(y)
    lib = _lib.load()
    b, n = y.shape
    mode, scal, lt = _lam1d(lam, y)
    stride = y.stride(0) if b > 1 else n
    x = torch.empty_like(y)
    if x.stride() != y.stride():
        x = torch.empty_strided(y.shape, y.stride(), device=y.device, dtype=y.dtype)
    mw = lib.tv1d_mask_words(n)
    mask = torch.empty((b, max(mw, 1)), device=y.device, dtype=torch.int32) if need_mask else None
    it = torch.empty(b, device=y.device, dtype=torch.int32) if want_iters else None
    if warm_mask is not None:
        _require_cuda(warm_mask)
    if opts is not None:
        check(lib.tv1d_prox_fwd_ex(dt, _ptr(y), _ptr(x), b, n, stride, _ptr(lt), mode, scal, _ptr(warm_mask),
                                   _ptr(mask), _ptr(it), _opts_ref(opts), _stream(y)), "tv1d_prox_fwd_ex")
    elif warm_mask is not None:
        check(lib.tv1d_prox_fwd_warm(dt, _ptr(y), _ptr(x), b, n, stride, _ptr(lt), mode, scal,
                                     _ptr(warm_mask), _ptr(mask), _ptr(it), _stream(y)), "tv1d_prox_fwd_warm")
    else:
        check(lib.tv1d_prox_fwd(dt, _ptr(y), _ptr(x), b, n, stride, _ptr(lt), mode, scal,
                                _ptr(mask), _ptr(it), _stream(y)), "tv1d_prox_fwd")
    return x, mask, it


def tv1d_bwd(grad_x: torch.Tensor, mask: torch.Tensor, lam_mode: int, want_lam: bool = True):
    """VJP of tv1d_fwd.  Returns (grad_y, grad_lam or None); grad_lam shape follows lam_mode."""
    _require_cuda(grad_x, mask)
    g = _rows(grad_x)
    dt = _dtype_code(g)
    lib = _lib.load()
    b, n = g.shape
    stride = g.stride(0) if b > 1 else n
    gy = torch.empty_strided(g.shape, g.stride(), device=g.device, dtype=g.dtype)
    glam = None
    if want_lam:
        if lam_mode == _lib.LAM_SCALAR:
            glam = torch.empty(1, device=g.device, dtype=g.dtype)
        elif lam_mode == _lib.LAM_PER_ROW:
            glam = torch.empty(b, device=g.device, dtype=g.dtype)
        else:
            glam = torch.zeros((b, stride), device=g.device, dtype=g.dtype)
    wsb = lib.tv1d_bwd_workspace_bytes(dt, b, lam_mode)
    ws = torch.empty(max(wsb, 1), device=g.device, dtype=torch.uint8)
    check(lib.tv1d_prox_bwd(dt, _ptr(g), _ptr(mask), _ptr(gy), _ptr(glam), b, n, stride, lam_mode,
                            _ptr(ws), _stream(g)), "tv1d_prox_bwd")
    if glam is not None and lam_mode == _lib.LAM_PER_EDGE:
        glam = glam[:, : max(n - 1, 0)]
    return gy, glam


class TV1DProx(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y, lam_t, lam_scalar):
        lam = lam_scalar if lam_t is None else lam_t
        x, mask, _ = tv1d_fwd(y, lam, need_mask=True)
        mode, _, _ = _lam1d(lam, _rows(y))
        ctx.save_for_backward(mask)
        ctx.mode = mode
        ctx.lam_shape = None if lam_t is None else lam_t.shape
        ctx.lam_device = None if lam_t is None else lam_t.device
        ctx.lam_dtype = None if lam_t is None else lam_t.dtype
        return x

    @staticmethod
    def backward(ctx, gx):
        (mask,) = ctx.saved_tensors
        need_lam = ctx.needs_input_grad[1]
        gy, gl = tv1d_bwd(gx.contiguous(), mask, ctx.mode, want_lam=need_lam)
        if need_lam and gl is not None and ctx.lam_shape is not None:
            gl = _lam_grad_like(gl, ctx.lam_shape, ctx.lam_device, ctx.lam_dtype)
        return gy, (gl if need_lam else None), None


def _lam_grad_like(gl: torch.Tensor, shape, device, dtype) -> torch.Tensor:
    """The lambda gradient in the caller's lambda layout: per-edge lambda given as
    [batch, n] or [batch, pitch] gets zeros beyond edge n-2 (those entries are not used),
    and the gradient lives on lambda's own device and dtype."""
    shape = torch.Size(shape)
    if gl.numel() != shape.numel():
        full = torch.zeros(shape, device=gl.device, dtype=gl.dtype)
        m = min(full.shape[-1], gl.shape[-1])
        full[..., :m] = gl.reshape(full.shape[0], -1)[:, :m]
        gl = full
    return gl.reshape(shape).to(device=device, dtype=dtype)


def tv1d(y: torch.Tensor, lam) -> torch.Tensor:
    """Differentiable batched 1D TV prox x = argmin 1/2||x-y||^2 + lam ||Dx||_1 (Eq. 1)."""
    if torch.is_tensor(lam):
        return TV1DProx.apply(y, lam, 0.0)
    return TV1DProx.apply(y, None, float(lam))


# ------------------------------------------------------------------------- 2D
def _lam2d(lam, X: torch.Tensor):
    N, C = X.shape[0], X.shape[1]
    if not torch.is_tensor(lam):
        return _lib.LAM_SCALAR, float(lam), None
    lam = lam.to(device=X.device, dtype=X.dtype)
    if lam.dim() == 0:
        return _lib.LAM_SCALAR, float(lam.item()), None
    if lam.numel() == C and (lam.dim() == 1 or lam.dim() == 2 and lam.shape[0] == 1):
        return _lib.LAM_PER_CHANNEL, 0.0, lam.reshape(C).contiguous()
    if lam.numel() == N * C:
        return _lib.LAM_PER_PLANE, 0.0, lam.reshape(N * C).contiguous()
    raise ValueError("tvprox: 2D lam must be a float, [C] or [N, C]")


def tv2d_fwd(X: torch.Tensor, lam, iters: int = 4, training: bool = True, want_iters: bool = False, opts=None,
             out: torch.Tensor = None):
    """Returns (Y, saved or None, line_iters or None).  opts: optional make_options(...);
    out: optional output tensor (may be X itself: in-place)."""
    _require_cuda(X)
    if X.dim() != 4:
        raise ValueError("tvprox: 2D input must be NCHW")
    X = X.contiguous()
    dt = _dtype_code(X)
    lib = _lib.load()
    N, C, H, W = X.shape
    mode, scal, lt = _lam2d(lam, X)
    if out is not None:
        _require_cuda(out)
        if out.shape != X.shape or out.dtype != X.dtype or not out.is_contiguous():
            raise ValueError("tvprox: out must be a contiguous tensor like X")
    Y = torch.empty_like(X) if out is None else out
    saved = None
    if training:
        sb = lib.tv2d_saved_bytes(N, C, H, W, iters)
        saved = torch.empty(max(sb // 4, 1), device=X.device, dtype=torch.int32)
    wsb = lib.tv2d_workspace_bytes(dt, N, C, H, W, iters)
    ws = torch.empty(max(wsb, 1), device=X.device, dtype=torch.uint8)
    it = torch.empty(2 * iters, device=X.device, dtype=torch.int32) if want_iters else None
    if opts is not None:
        check(lib.tv2d_prox_fwd_ex(dt, _ptr(X), _ptr(Y), N, C, H, W, _ptr(lt), mode, scal, int(iters),
                                   _ptr(saved), _ptr(ws), _ptr(it), _opts_ref(opts), _stream(X)), "tv2d_prox_fwd_ex")
    else:
        check(lib.tv2d_prox_fwd(dt, _ptr(X), _ptr(Y), N, C, H, W, _ptr(lt), mode, scal, int(iters),
                                _ptr(saved), _ptr(ws), _ptr(it), _stream(X)), "tv2d_prox_fwd")
    return Y, saved, it


def tv2d_bwd(grad_Y: torch.Tensor, saved: torch.Tensor, lam_mode: int, iters: int, want_lam: bool = True,
             opts=None, out: torch.Tensor = None):
    """Returns (grad_X, grad_lam or None).  out: optional grad_X tensor (may be grad_Y: in-place)."""
    _require_cuda(grad_Y, saved)
    G = grad_Y.contiguous()
    dt = _dtype_code(G)
    lib = _lib.load()
    N, C, H, W = G.shape
    if out is not None:
        _require_cuda(out)
        if out.shape != G.shape or out.dtype != G.dtype or not out.is_contiguous():
            raise ValueError("tvprox: out must be a contiguous tensor like grad_Y")
    GX = torch.empty_like(G) if out is None else out
    glam = None
    if want_lam:
        cnt = {_lib.LAM_SCALAR: 1, _lib.LAM_PER_CHANNEL: C, _lib.LAM_PER_PLANE: N * C}[lam_mode]
        glam = torch.empty(max(cnt, 1), device=G.device, dtype=G.dtype)
    wsb = lib.tv2d_workspace_bytes(dt, N, C, H, W, iters)
    ws = torch.empty(max(wsb, 1), device=G.device, dtype=torch.uint8)
    if opts is not None:
        check(lib.tv2d_prox_bwd_ex(dt, _ptr(G), _ptr(saved), _ptr(GX), _ptr(glam), N, C, H, W, lam_mode,
                                   int(iters), _ptr(ws), _opts_ref(opts), _stream(G)), "tv2d_prox_bwd_ex")
    else:
        check(lib.tv2d_prox_bwd(dt, _ptr(G), _ptr(saved), _ptr(GX), _ptr(glam), N, C, H, W, lam_mode,
                                int(iters), _ptr(ws), _stream(G)), "tv2d_prox_bwd")
    return GX, glam


class TV2DProx(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, lam_t, lam_scalar, iters):
        lam = lam_scalar if lam_t is None else lam_t
        Y, saved, _ = tv2d_fwd(X, lam, iters, training=True)
        mode, _, _ = _lam2d(lam, X)
        ctx.save_for_backward(saved)
        ctx.mode, ctx.iters = mode, iters
        ctx.lam_shape = None if lam_t is None else lam_t.shape
        ctx.lam_device = None if lam_t is None else lam_t.device
        ctx.lam_dtype = None if lam_t is None else lam_t.dtype
        return Y

    @staticmethod
    def backward(ctx, gY):
        (saved,) = ctx.saved_tensors
        need_lam = ctx.needs_input_grad[1]
        gX, gl = tv2d_bwd(gY, saved, ctx.mode, ctx.iters, want_lam=need_lam)
        if need_lam and gl is not None and ctx.lam_shape is not None:
            gl = gl.reshape(ctx.lam_shape).to(device=ctx.lam_device, dtype=ctx.lam_dtype)
        return gX, (gl if need_lam else None), None, None


def tv2d(X: torch.Tensor, lam, iters: int = 4) -> torch.Tensor:
    """Differentiable anisotropic 2D TV prox by K = iters Proximal Dykstra iterations (Alg. 1)."""
    if torch.is_tensor(lam):
        return TV2DProx.apply(X, lam, 0.0, int(iters))
    return TV2DProx.apply(X, None, float(lam), int(iters))


# --------------------------------------------------- TV layer pieces (NEXT f1)
def tv2d_lines_fwd(X: torch.Tensor, lam, axis: int, need_mask: bool = True):
    """Rows-only (axis 0) / columns-only (axis 1) spatial mode.  Returns (Y, mask)."""
    _require_cuda(X)
    X = X.contiguous()
    dt = _dtype_code(X)
    lib = _lib.load()
    N, C, H, W = X.shape
    mode, scal, lt = _lam2d(lam, X)
    Y = torch.empty_like(X)
    L, n = (H, W) if axis == 0 else (W, H)
    mask = None
    if need_mask:
        mw = lib.tv1d_mask_words(n)
        mask = torch.empty((N * C * L, max(mw, 1)), device=X.device, dtype=torch.int32)
    check(lib.tv2d_lines_fwd(dt, _ptr(X), _ptr(Y), N, C, H, W, _ptr(lt), mode, scal, int(axis), _ptr(mask),
                             _stream(X)), "tv2d_lines_fwd")
    return Y, mask


def tv2d_lines_bwd(grad_Y: torch.Tensor, mask: torch.Tensor, lam_mode: int, axis: int, want_lam: bool = True):
    _require_cuda(grad_Y, mask)
    G = grad_Y.contiguous()
    dt = _dtype_code(G)
    lib = _lib.load()
    N, C, H, W = G.shape
    GX = torch.empty_like(G)
    glam = None
    if want_lam:
        cnt = {_lib.LAM_SCALAR: 1, _lib.LAM_PER_CHANNEL: C, _lib.LAM_PER_PLANE: N * C}[lam_mode]
        glam = torch.empty(max(cnt, 1), device=G.device, dtype=G.dtype)
    ws = torch.empty(max(lib.tv2d_lines_workspace_bytes(dt, N, C, H, W, int(axis)), 1), device=G.device,
                     dtype=torch.uint8)
    check(lib.tv2d_lines_bwd(dt, _ptr(G), _ptr(mask), _ptr(GX), _ptr(glam), N, C, H, W, lam_mode, int(axis),
                             _ptr(ws), _stream(G)), "tv2d_lines_bwd")
    return GX, glam


class TVLinesProx(torch.autograd.Function):
    @staticmethod
    def forward(ctx, X, lam_t, lam_scalar, axis):
        lam = lam_scalar if lam_t is None else lam_t
        Y, mask = tv2d_lines_fwd(X, lam, axis)
        mode, _, _ = _lam2d(lam, X)
        ctx.save_for_backward(mask)
        ctx.mode, ctx.axis = mode, axis
        ctx.lam_shape = None if lam_t is None else lam_t.shape
        ctx.lam_device = None if lam_t is None else lam_t.device
        ctx.lam_dtype = None if lam_t is None else lam_t.dtype
        return Y

    @staticmethod
    def backward(ctx, gY):
        (mask,) = ctx.saved_tensors
        need_lam = ctx.needs_input_grad[1]
        gX, gl = tv2d_lines_bwd(gY, mask, ctx.mode, ctx.axis, want_lam=need_lam)
        if need_lam and gl is not None and ctx.lam_shape is not None:
            gl = gl.reshape(ctx.lam_shape).to(device=ctx.lam_device, dtype=ctx.lam_dtype)
        return gX, (gl if need_lam else None), None, None


def tv2d_lines(X: torch.Tensor, lam, axis: int) -> torch.Tensor:
    if torch.is_tensor(lam):
        return TVLinesProx.apply(X, lam, 0.0, int(axis))
    return TVLinesProx.apply(X, None, float(lam), int(axis))


def softplus_fwd(t: torch.Tensor) -> torch.Tensor:
    _require_cuda(t)
    t = t.contiguous()
    out = torch.empty_like(t)
    check(_lib.load().tvp_softplus_fwd(_dtype_code(t), _ptr(t), _ptr(out), t.numel(), _stream(t)), "tvp_softplus_fwd")
    return out


def softplus_bwd(t: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    _require_cuda(t, g)
    t, g = t.contiguous(), g.contiguous().to(t.dtype)
    out = torch.empty_like(t)
    check(_lib.load().tvp_softplus_bwd(_dtype_code(t), _ptr(t), _ptr(g), _ptr(out), t.numel(), _stream(t)),
          "tvp_softplus_bwd")
    return out


def axpby_(x, y: torch.Tensor, a: float, b: float) -> torch.Tensor:
    """In place: y <- a x + b y (one kernel)."""
    _require_cuda(y)
    if x is not None:
        _require_cuda(x)
        x = x.contiguous()
    assert y.is_contiguous()
    check(_lib.load().tvp_axpby(_dtype_code(y), _ptr(x), _ptr(y), float(a), float(b), y.numel(), _stream(y)),
          "tvp_axpby")
    return y


def unpack_mask(mask: torch.Tensor, n: int) -> torch.Tensor:
    """[lines, words] int32 -> [lines, n-1] uint8 2-bit codes (host-side helper for tests/diagnostics)."""
    m = mask.to(torch.int64) & 0xFFFFFFFF
    lines = m.shape[0]
    e = torch.arange(max(n - 1, 0), device=m.device)
    return ((m[:, e // 16] >> (2 * (e % 16))) & 3).to(torch.uint8).reshape(lines, -1)
