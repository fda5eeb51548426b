"""CPU oracle for arXiv 2204.03643 (TV proximity operators) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2204_03643_b200``) never imports it, and it shares no code with the
CUDA library.  See ``oracle/tvref.c`` for the passage each function follows
(Eq. 1, Eq. 7-8, Algorithm 1) and DESIGN.md for the readings.

Everything here is fp64 numpy on the host; the arithmetic lives in
``tvref.c`` (plain C99, compiled with gcc into ``liboracle.so``) and in the
small numpy helpers below (dense Eq. 8, KKT certificate, objective).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tvref.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile tvref.c with gcc (plain -O2, no fast-math) into liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        cmd = ["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-pthread", "-fno-fast-math",
               "-D_POSIX_C_SOURCE=200809L", _SRC, "-o", tmp, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _get():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            i64, dp, i8p = ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p
            lib.tvref_prox1d.argtypes = [i64, dp, ctypes.c_double, dp]
            lib.tvref_prox1d_edges.argtypes = [i64, dp, dp, dp]
            lib.tvref_codes.argtypes = [i64, dp, dp, ctypes.c_double, i8p, i8p]
            lib.tvref_codes.restype = None
            lib.tvref_bwd1d.argtypes = [i64, i8p, i8p, dp, dp, dp, dp]
            lib.tvref_bwd1d.restype = None
            lib.tvref_prox2d.argtypes = [i64, i64, dp, ctypes.c_double, ctypes.c_int, dp,
                                         i8p, i8p, i8p, i8p]
            lib.tvref_bwd2d.argtypes = [i64, i64, ctypes.c_int, i8p, i8p, i8p, i8p, dp, dp, dp]
            lib.tvref_prox1d_batch.argtypes = [i64, i64, dp, dp, ctypes.c_int, dp, i8p, i8p,
                                               ctypes.c_int]
            lib.tvref_bwd1d_batch.argtypes = [i64, i64, i8p, i8p, dp, dp, dp, ctypes.c_int,
                                              ctypes.c_int]
            lib.tvref_prox2d_batch.argtypes = [i64, i64, i64, dp, dp, ctypes.c_int, dp,
                                               i8p, i8p, i8p, i8p, ctypes.c_int]
            lib.tvref_bwd2d_batch.argtypes = [i64, i64, i64, ctypes.c_int, i8p, i8p, i8p, i8p,
                                              dp, dp, dp, ctypes.c_int]
            lib.tvref_prox2d_batch_ex.argtypes = [i64, i64, i64, dp, dp, ctypes.c_int, dp,
                                                  i8p, i8p, i8p, i8p, dp, dp, ctypes.c_int]
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i8(a):
    return np.ascontiguousarray(a, dtype=np.int8)


# --------------------------------------------------------------------------- 1D
def prox1d(y, lam):
    """Exact 1D TV prox (Eq. 1).  lam: scalar, or array of n-1 per-edge weights."""
    y = _f64(y)
    n = y.shape[0]
    x = np.empty_like(y)
    if n == 0:
        return x
    if np.ndim(lam) == 0:
        st = _get().tvref_prox1d(n, _p(y), float(lam), _p(x))
    else:
        le = _f64(lam)
        assert le.shape == (max(n - 1, 0),)
        st = _get().tvref_prox1d_edges(n, _p(y), _p(le) if n > 1 else None, _p(x))
    if st:
        raise MemoryError("tvref prox1d failed")
    return x


def codes(x, lam):
    """(brk, sgn) of a 1D solution: jump edges and their signs (support of D x)."""
    x = _f64(x)
    n = x.shape[0]
    m = max(n - 1, 0)
    brk = np.zeros(m, np.int8)
    sgn = np.zeros(m, np.int8)
    if m:
        if np.ndim(lam) == 0:
            _get().tvref_codes(n, _p(x), None, float(lam), _p(brk), _p(sgn))
        else:
            le = _f64(lam)
            _get().tvref_codes(n, _p(x), _p(le), 0.0, _p(brk), _p(sgn))
    return brk, sgn


def bwd1d(brk, sgn, g):
    """Segment-mean VJP (Eq. 7-8 under O12).  Returns (grad_y, grad_lam_edges, grad_lam_total)."""
    g = _f64(g)
    n = g.shape[0]
    brk, sgn = _i8(brk), _i8(sgn)
    gy = np.empty_like(g)
    ge = np.zeros(max(n - 1, 0))
    gt = np.zeros(1)
    if n:
        _get().tvref_bwd1d(n, _p(brk), _p(sgn), _p(g), _p(gy), _p(ge), _p(gt))
    return gy, ge, float(gt[0])


def prox1d_batch(y, lam, per_edge=False, nthreads=1, with_codes=True):
    """Rows of y [batch, n] independently; lam: [batch] (per row) or [batch, n-1] (per edge)."""
    y = _f64(y)
    b, n = y.shape
    lam = _f64(lam)
    x = np.empty_like(y)
    m = max(n - 1, 0)
    brk = np.zeros((b, m), np.int8) if with_codes else None
    sgn = np.zeros((b, m), np.int8) if with_codes else None
    st = _get().tvref_prox1d_batch(b, n, _p(y), _p(lam), int(per_edge), _p(x),
                                   _p(brk), _p(sgn), int(nthreads))
    if st:
        raise MemoryError("tvref prox1d_batch failed")
    return x, brk, sgn


def bwd1d_batch(brk, sgn, g, per_edge=False, nthreads=1):
    g = _f64(g)
    b, n = g.shape
    gy = np.empty_like(g)
    gl = np.zeros((b, max(n - 1, 0))) if per_edge else np.zeros(b)
    brk, sgn = _i8(brk), _i8(sgn)      # keep the converted copies alive across the call
    _get().tvref_bwd1d_batch(b, n, _p(brk), _p(sgn), _p(g), _p(gy), _p(gl),
                             int(per_edge), int(nthreads))
    return gy, gl


# --------------------------------------------------------------------------- 2D
def prox2d(X, lam, K):
    """Algorithm 1 literal.  Returns (Y, (rbrk, rsgn, cbrk, csgn))."""
    X = _f64(X)
    H, W = X.shape
    Y = np.empty_like(X)
    rb = np.zeros((K, H, max(W - 1, 0)), np.int8)
    rs = np.zeros_like(rb)
    cb = np.zeros((K, W, max(H - 1, 0)), np.int8)
    cs = np.zeros_like(cb)
    st = _get().tvref_prox2d(H, W, _p(X), float(lam), int(K), _p(Y), _p(rb), _p(rs), _p(cb), _p(cs))
    if st:
        raise MemoryError("tvref prox2d failed")
    return Y, (rb, rs, cb, cs)


def bwd2d(segs, G, K):
    """Reverse mode through K iterations of Algorithm 1.  Returns (grad_X, grad_lam)."""
    rb, rs, cb, cs = (_i8(s) for s in segs)
    G = _f64(G)
    H, W = G.shape
    GX = np.empty_like(G)
    gl = np.zeros(1)
    st = _get().tvref_bwd2d(H, W, int(K), _p(rb), _p(rs), _p(cb), _p(cs), _p(G), _p(GX), _p(gl))
    if st:
        raise MemoryError("tvref bwd2d failed")
    return GX, float(gl[0])


def prox2d_batch(X, lam, K, nthreads=1, with_codes=True, with_jumps=False):
    """Planes X [P, H, W], lam [P].  Returns (Y, segs), or (Y, segs, (rjmp, cjmp)) with
    with_jumps: the jumps out[e+1] - out[e] of every 1D pass output, [P][K][lines][n-1]."""
    X = _f64(X)
    P, H, W = X.shape
    lam = _f64(lam)
    Y = np.empty_like(X)
    if with_codes:
        rb = np.zeros((P, K, H, max(W - 1, 0)), np.int8)
        rs = np.zeros_like(rb)
        cb = np.zeros((P, K, W, max(H - 1, 0)), np.int8)
        cs = np.zeros_like(cb)
    else:
        rb = rs = cb = cs = None
    rj = np.zeros((P, K, H, max(W - 1, 0))) if with_jumps else None
    cj = np.zeros((P, K, W, max(H - 1, 0))) if with_jumps else None
    st = _get().tvref_prox2d_batch_ex(P, H, W, _p(X), _p(lam), int(K), _p(Y), _p(rb), _p(rs),
                                      _p(cb), _p(cs), _p(rj), _p(cj), int(nthreads))
    if st:
        raise MemoryError("tvref prox2d_batch failed")
    if with_jumps:
        return Y, (rb, rs, cb, cs), (rj, cj)
    return Y, (rb, rs, cb, cs)


def bwd2d_batch(segs, G, K, nthreads=1):
    rb, rs, cb, cs = (_i8(s) for s in segs)
    G = _f64(G)
    P, H, W = G.shape
    GX = np.empty_like(G)
    gl = np.zeros(P)
    st = _get().tvref_bwd2d_batch(P, H, W, int(K), _p(rb), _p(rs), _p(cb), _p(cs), _p(G),
                                  _p(GX), _p(gl), int(nthreads))
    if st:
        raise MemoryError("tvref bwd2d_batch failed")
    return GX, gl


# --------------------------------------------------------------- plain numpy checks
def diff(z):
    """(D z)_i = z_{i+1} - z_i  (reading O2)."""
    return np.diff(np.asarray(z, dtype=np.float64))


def objective1d(x, y, lam):
    """Eq. 1 objective 1/2||x - y||^2 + sum_i lam_i |x_{i+1} - x_i|."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    return 0.5 * np.sum((x - y) ** 2) + np.sum(np.asarray(lam) * np.abs(np.diff(x)))
