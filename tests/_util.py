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
