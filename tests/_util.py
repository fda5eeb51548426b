"""Test-side helpers (independent of both the oracle's arithmetic and the CUDA path)."""
import numpy as np

TOL = {"f32": 1e-4, "f64": 1e-9}     # north_star: max-abs error relative to the input range


def unpack_codes(mask_words, n):
    """uint32 words [lines, mw] -> int8 codes [lines, n-1] (2 bits per edge, include/tvprox.h)."""
    m = np.asarray(mask_words).astype(np.uint32)
    lines = m.shape[0]
    e = np.arange(max(n - 1, 0))
    if e.size == 0:
        return np.zeros((lines, 0), np.int8)
    return np.ascontiguousarray(((m[:, e // 16] >> (2 * (e % 16)).astype(np.uint32)) & 3).astype(np.int8))


def codes_to_brk_sgn(codes):
    codes = np.asarray(codes)
    brk = np.ascontiguousarray((codes != 0).astype(np.int8))
    sgn = np.ascontiguousarray(np.where(codes == 1, 1, np.where(codes == 2, -1, 0)).astype(np.int8))
    return brk, sgn


def brk_sgn_to_codes(brk, sgn, lam_zero=None):
    c = np.where(sgn > 0, 1, np.where(sgn < 0, 2, 0))
    if lam_zero is not None:
        c = np.where((brk != 0) & (sgn == 0), 3, c)
    return c.astype(np.int8)


def rel_err(a, b, ref_range):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)) / max(ref_range, 1e-300))


def rng_range(x):
    x = np.asarray(x, np.float64)
    return float(x.max() - x.min()) if x.size else 0.0


def _spread(taint, brk):
    """Any tainted sample of a segment (breaks brk [L, n-1] != 0) taints the whole segment."""
    L, n = taint.shape
    if n == 0:
        return taint.copy()
    seg = np.zeros((L, n), np.int64)
    if n > 1:
        seg[:, 1:] = np.cumsum(brk != 0, axis=1)
    ids = seg + (np.arange(L, dtype=np.int64)[:, None] * n)
    cnt = np.bincount(ids.ravel(), weights=taint.ravel().astype(np.float64), minlength=L * n)
    return cnt[ids] > 0


def taint_2d(gpu_segs, ref_segs, H, W, K):
    """Pixels of each plane whose 2D adjoint (reverse mode through Alg. 1, a-14) can depend
    on a mask disagreement between two segmentations (reading O13 (ii) in 2D).

    segs = (rbrk [P][K][H][W-1], rsgn, cbrk [P][K][W][H-1], csgn).  Reverse order
    k = K..1: column adjoint, then row adjoint.  A pass seeds both samples of every edge
    whose break flag differs, and the output of a segment-mean pass at a pixel can differ
    when that pixel's segment under EITHER segmentation holds a tainted input.
    Returns a bool array [P, H, W]."""
    grb, _, gcb, _ = gpu_segs
    orb, _, ocb, _ = ref_segs
    P = grb.shape[0]
    out = np.zeros((P, H, W), bool)
    for p in range(P):
        t = np.zeros((H, W), bool)
        for k in range(K - 1, -1, -1):
            # column adjoint k (lines = columns)
            tc = t.T.copy()
            if H > 1:
                d = gcb[p, k] != ocb[p, k]
                tc[:, :-1] |= d
                tc[:, 1:] |= d
            tc = _spread(tc, gcb[p, k]) | _spread(tc, ocb[p, k])
            t = tc.T.copy()
            # row adjoint k
            if W > 1:
                d = grb[p, k] != orb[p, k]
                t[:, :-1] |= d
                t[:, 1:] |= d
            t = _spread(t, grb[p, k]) | _spread(t, orb[p, k])
        out[p] = t
    return out
