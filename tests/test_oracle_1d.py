"""Pins for the 1D oracle (oracle/tvref.c) against what the paper and the mathematics fix.

Every check here is independent of the oracle's own arithmetic: brute-force
enumeration of the finite KKT sign patterns, closed forms, the KKT optimality
certificate of Eq. 1, the paper's lam = 0 identity, SPEC worked
examples, a projected-gradient dual solver, dense Eq. 8, and
central finite differences.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------- independent helpers
def brute_force_prox(y, lam):
    """Enumerate s in {-1,0,+1}^(n-1) (the possible signs of D x).  For each pattern the
    KKT conditions of Eq. 1 fix x: segments are runs joined by s=0 edges, a segment
    [a,b) takes mean(y) + (lam_{b-1} s_{b-1} - lam_{a-1} s_{a-1}) / (b-a).  Keep the
    patterns whose jumps have exactly the signs s and whose fused duals are feasible.
    Returns the list of all surviving x (all equal: the prox is unique)."""
    y = np.asarray(y, np.float64)
    n = len(y)
    lam = np.broadcast_to(np.asarray(lam, np.float64), (max(n - 1, 0),))
    sols = []
    for s in itertools.product((-1, 0, 1), repeat=n - 1):
        x = np.empty(n)
        a = 0
        ok = True
        while a < n:
            b = a + 1
            while b < n and s[b - 1] == 0:
                b += 1
            right = lam[b - 1] * s[b - 1] if b < n else 0.0
            left = lam[a - 1] * s[a - 1] if a > 0 else 0.0
            x[a:b] = y[a:b].mean() + (right - left) / (b - a)
            a = b
        for e in range(n - 1):
            d = x[e + 1] - x[e]
            if s[e] != 0 and not (np.sign(d) == s[e] and abs(d) > 1e-12):
                ok = False
                break
        if not ok:
            continue
        u = np.cumsum(x - y)[:-1]
        if np.all(np.abs(u) <= lam + 1e-12):
            sols.append(x)
    return sols


def kkt_residual(x, y, lam):
    """Max violation of the optimality conditions of Eq. 1 for candidate x:
    u = cumsum(x - y) is the dual (x = y - D^T u); need u_{n-1} = 0, |u_i| <= lam_i and
    u_i = lam_i sign(x_{i+1} - x_i) wherever x_{i+1} != x_i."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    n = len(y)
    lam = np.broadcast_to(np.asarray(lam, np.float64), (max(n - 1, 0),))
    c = np.cumsum(x - y)
    r = abs(c[-1])
    if n > 1:
        u = c[:-1]
        r = max(r, np.max(np.maximum(np.abs(u) - lam, 0.0)))
        d = np.diff(x)
        jump = d != 0
        if np.any(jump):
            r = max(r, np.max(np.abs(u[jump] - lam[jump] * np.sign(d[jump]))))
    return r


def pgd_dual(y, lam, iters=100000, step=0.25):
    """Projected gradient ascent on the dual Eq. 5, step 1/||DD^T|| <= 1/4
    (S:527-535).  Independent, approximate."""
    y = np.asarray(y, np.float64)
    u = np.zeros(len(y) - 1)
    for _ in range(iters):
        x = y.copy()
        x[:-1] += u
        x[1:] -= u
        u = np.clip(u + step * np.diff(x), -lam, lam)
    x = y.copy()
    x[:-1] += u
    x[1:] -= u
    return x


# ----------------------------------------------------------------- worked examples
def test_spec_two_point_examples():
    # S:240-242
    assert np.array_equal(oracle.prox1d([0.0, 2.0], 0.5), [0.5, 1.5])
    assert np.array_equal(oracle.prox1d([0.0, 2.0], 5.0), [1.0, 1.0])


def test_two_point_closed_form():
    rng = np.random.default_rng(1)
    for _ in range(200):
        y = rng.standard_normal(2) * 3
        lam = rng.uniform(0, 3)
        d = y[1] - y[0]
        lp = min(lam, abs(d) / 2)
        exp = np.array([y[0] + np.sign(d) * lp, y[1] - np.sign(d) * lp])
        np.testing.assert_allclose(oracle.prox1d(y, lam), exp, atol=1e-14)


def test_golden_vectors():
    with open(os.path.join(GOLDEN, "tv1d.json")) as f:
        gold = json.load(f)
    for case in gold["forward"]:
        # the stored value is itself certified optimal for Eq. 1 (independent of the oracle)
        assert kkt_residual(case["x"], case["y"], case["lam"]) < 1e-12, case["cite"]
        x = oracle.prox1d(case["y"], case["lam"])
        np.testing.assert_allclose(x, case["x"], atol=1e-12, err_msg=case["cite"])


def test_unit_step_closed_form():
    # step 0 -> h at p: one jump with values lam/p and h - lam/(n-p) while lam < h p (n-p)/n,
    # else the mean (derived from the KKT conditions, SURVEY 8(c) pins).
    for n in (2, 5, 8, 33, 64, 1000):
        for p in sorted({1, n // 2, n - 1}):
            if p <= 0 or p >= n:
                continue
            for h in (1.0, -2.5):
                y = np.zeros(n)
                y[p:] = h
                thr = abs(h) * p * (n - p) / n
                for lam in (0.1 * thr, 0.5 * thr, 0.999 * thr, thr, 1.5 * thr):
                    x = oracle.prox1d(y, lam)
                    if lam < thr:
                        s = np.sign(h)
                        exp = np.concatenate([np.full(p, s * lam / p), np.full(n - p, h - s * lam / (n - p))])
                    else:
                        exp = np.full(n, y.mean())
                    np.testing.assert_allclose(x, exp, atol=1e-12 * max(1, abs(h) * n))


def test_lambda_max_closed_form():
    rng = np.random.default_rng(2)
    for _ in range(100):
        n = rng.integers(2, 80)
        y = rng.standard_normal(n)
        lmax = np.max(np.abs(np.cumsum(y - y.mean())[:-1]))
        x = oracle.prox1d(y, lmax * 1.0000001)
        np.testing.assert_allclose(x, np.full(n, y.mean()), atol=1e-12)
        x = oracle.prox1d(y, lmax * 0.99)
        assert np.ptp(x) > 0


# ----------------------------------------------------------------- brute force / KKT
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8])
def test_brute_force_small(n):
    rng = np.random.default_rng(100 + n)
    for trial in range(40):
        y = rng.standard_normal(n) * rng.choice([0.3, 1.0, 3.0])
        lam = rng.choice([0.05, 0.3, 1.0, 4.0])
        sols = brute_force_prox(y, lam)
        assert len(sols) >= 1
        x = oracle.prox1d(y, lam)
        for s in sols:
            np.testing.assert_allclose(x, s, atol=1e-12)


@pytest.mark.parametrize("n", [2, 3, 5, 7])
def test_brute_force_per_edge(n):
    rng = np.random.default_rng(200 + n)
    for trial in range(40):
        y = rng.standard_normal(n)
        lam = rng.uniform(0.0, 1.5, size=n - 1)
        lam[rng.random(n - 1) < 0.15] = 0.0
        sols = brute_force_prox(y, lam)
        x = oracle.prox1d(y, lam)
        for s in sols:
            np.testing.assert_allclose(x, s, atol=1e-12)


def test_kkt_certificate_large():
    rng = np.random.default_rng(3)
    for n in (100, 1024, 4096):
        for kind in ("normal", "step"):
            y = rng.standard_normal(n) if kind == "normal" else (np.arange(n) >= n // 2) + 0.1 * rng.standard_normal(n)
            for lam in (0.01, 0.3, 1.0, 10.0):
                x = oracle.prox1d(y, lam)
                assert kkt_residual(x, y, lam) < 1e-9
                le = rng.uniform(0.0, 2 * lam, size=n - 1)
                xe = oracle.prox1d(y, le)
                assert kkt_residual(xe, y, le) < 1e-9


def test_per_edge_uniform_matches_scalar():
    rng = np.random.default_rng(4)
    for _ in range(50):
        n = int(rng.integers(2, 300))
        y = rng.standard_normal(n)
        lam = float(rng.uniform(0.01, 3))
        np.testing.assert_allclose(oracle.prox1d(y, np.full(n - 1, lam)), oracle.prox1d(y, lam), atol=1e-11)


def test_per_edge_zero_weight_decouples():
    # lam_e = 0 removes the coupling across edge e: the problem splits in two.
    rng = np.random.default_rng(5)
    for _ in range(30):
        n = int(rng.integers(4, 60))
        e = int(rng.integers(0, n - 1))
        y = rng.standard_normal(n)
        le = rng.uniform(0.1, 1.0, size=n - 1)
        le[e] = 0.0
        x = oracle.prox1d(y, le)
        left = oracle.prox1d(y[: e + 1], le[:e]) if e > 0 else y[:1]
        right = oracle.prox1d(y[e + 1:], le[e + 1:]) if e + 1 < n - 1 else y[e + 1:]
        np.testing.assert_allclose(x, np.concatenate([left, right]), atol=1e-12)


def test_pgd_dual_agreement():
    rng = np.random.default_rng(6)
    for _ in range(6):
        n = int(rng.integers(3, 16))
        y = rng.standard_normal(n)
        lam = float(rng.choice([0.1, 0.5, 1.0]))
        np.testing.assert_allclose(oracle.prox1d(y, lam), pgd_dual(y, lam, iters=20000), atol=1e-6)


# ----------------------------------------------------------------- invariants
def test_lambda_zero_identity_bitwise():
    # lam = 0 is the identity
    rng = np.random.default_rng(7)
    y = rng.standard_normal(257)
    assert np.array_equal(oracle.prox1d(y, 0.0), y)
    assert np.array_equal(oracle.prox1d(y, np.zeros(256)), y)


def test_n1_and_constant():
    assert np.array_equal(oracle.prox1d([3.0], 2.0), [3.0])
    np.testing.assert_allclose(oracle.prox1d(np.full(17, 1.25), 0.7), np.full(17, 1.25), rtol=1e-15)


def test_invariants_random():
    rng = np.random.default_rng(8)
    for _ in range(100):
        n = int(rng.integers(2, 200))
        y = rng.standard_normal(n)
        lam = float(rng.uniform(0.01, 2))
        x = oracle.prox1d(y, lam)
        assert abs(x.sum() - y.sum()) < 1e-10 * n                   # sum preservation
        c = float(rng.standard_normal())
        np.testing.assert_allclose(oracle.prox1d(y + c, lam), x + c, atol=1e-11)   # translation
        y2 = y + 0.3 * rng.standard_normal(n)
        x2 = oracle.prox1d(y2, lam)
        assert np.linalg.norm(x - x2) <= np.linalg.norm(y - y2) + 1e-12            # nonexpansive
        x3 = oracle.prox1d(y, lam * 1.7)
        assert np.abs(np.diff(x3)).sum() <= np.abs(np.diff(x)).sum() + 1e-12       # TV monotone
        # optimality vs random feasible perturbations of the objective
        f0 = oracle.objective1d(x, y, lam)
        for _ in range(5):
            assert oracle.objective1d(x + 1e-3 * rng.standard_normal(n), y, lam) >= f0 - 1e-14


def test_piecewise_constant_exact_values():
    rng = np.random.default_rng(9)
    y = rng.standard_normal(500)
    x = oracle.prox1d(y, 1.0)
    brk, sgn = oracle.codes(x, 1.0)
    assert brk.sum() < 499       # fusion happened
    # values are exactly equal inside segments (codes read off by exact equality)
    assert np.all((np.diff(x) == 0) == (brk == 0))


# ----------------------------------------------------------------- backward
def dense_eq8(x):
    """Eq. 7-8 written out with dense matrices under reading O12."""
    x = np.asarray(x, np.float64)
    n = x.shape[0]
    dx = np.diff(x)
    L = np.tril(np.ones((n, n)))
    S = [0] + [i + 1 for i in range(n - 1) if dx[i] != 0.0]
    LS = L[:, S]
    M = LS @ np.linalg.inv(LS.T @ LS)
    J = M @ LS.T
    sg = np.array([0.0] + [np.sign(dx[s - 1]) for s in S[1:]])
    return J, -M @ sg


def test_spec_vjp_examples():
    # S:326-338 (sign from S:336, not the prose at S:333; reading O14)
    gy, _, _ = oracle.bwd1d([0], [0], [1.0, 0.0])
    assert np.array_equal(gy, [0.5, 0.5])
    gy, _, _ = oracle.bwd1d([0, 1], [0, 1], [2.0, 0.0, 7.0])
    assert np.array_equal(gy, [1.0, 1.0, 7.0])
    x = oracle.prox1d([0.0, 2.0], 0.5)
    b, s = oracle.codes(x, 0.5)
    _, _, gl = oracle.bwd1d(b, s, [1.0, 0.0])
    assert gl == 1.0
    _, _, gl = oracle.bwd1d(b, s, [1.0, 1.0])
    assert gl == 0.0


def test_golden_backward():
    with open(os.path.join(GOLDEN, "tv1d.json")) as f:
        gold = json.load(f)
    for case in gold["backward"]:
        x = oracle.prox1d(case["y"], case["lam"])
        b, s = oracle.codes(x, case["lam"])
        gy, _, gl = oracle.bwd1d(b, s, case["g"])
        np.testing.assert_allclose(gy, case["grad_y"], atol=1e-12, err_msg=case["cite"])
        assert abs(gl - case["grad_lam"]) < 1e-12


def test_dense_eq8_equals_segment_mean():
    rng = np.random.default_rng(10)
    for _ in range(60):
        n = int(rng.integers(1, 64))
        y = rng.standard_normal(n)
        lam = float(rng.uniform(0.05, 2))
        x = oracle.prox1d(y, lam)
        b, s = oracle.codes(x, lam)
        J, dl = dense_eq8(x)
        np.testing.assert_allclose(J, J.T, atol=1e-10)          # projector laws
        np.testing.assert_allclose(J @ J, J, atol=1e-10)
        assert abs(dl.sum()) < 1e-10                            # zero-sum dx/dlam
        g = rng.standard_normal(n)
        gy, ge, gl = oracle.bwd1d(b, s, g)
        np.testing.assert_allclose(gy, J.T @ g, atol=1e-10)
        assert abs(gl - dl @ g) < 1e-10
        assert abs(ge.sum() - gl) < 1e-10


def _nondegenerate(y, lam, margin=1e-3):
    x = oracle.prox1d(y, lam)
    lam_e = np.broadcast_to(np.asarray(lam, np.float64), (len(y) - 1,))
    u = np.cumsum(x - y)[:-1]
    d = np.diff(x)
    fused = d == 0
    if np.any(np.abs(d[~fused]) < margin):
        return False
    if np.any(np.abs(u[fused]) > lam_e[fused] - margin):
        return False
    return True


def test_finite_differences_scalar_and_edge():
    rng = np.random.default_rng(11)
    h = 1e-6
    done = 0
    for _ in range(200):
        n = int(rng.integers(2, 33))
        y = rng.standard_normal(n)
        lam = float(rng.choice([0.3, 1.0]))
        if not _nondegenerate(y, lam):
            continue
        x = oracle.prox1d(y, lam)
        b, s = oracle.codes(x, lam)
        g = rng.standard_normal(n)
        gy, ge, gl = oracle.bwd1d(b, s, g)
        fd = np.array([(g @ oracle.prox1d(y + h * np.eye(n)[i], lam) -
                        g @ oracle.prox1d(y - h * np.eye(n)[i], lam)) / (2 * h) for i in range(n)])
        np.testing.assert_allclose(gy, fd, atol=1e-6)
        fdl = (g @ oracle.prox1d(y, lam + h) - g @ oracle.prox1d(y, lam - h)) / (2 * h)
        assert abs(gl - fdl) < 1e-6
        le = np.full(n - 1, lam)
        fde = np.array([(g @ oracle.prox1d(y, le + h * np.eye(n - 1)[e]) -
                         g @ oracle.prox1d(y, le - h * np.eye(n - 1)[e])) / (2 * h) for e in range(n - 1)])
        np.testing.assert_allclose(ge, fde, atol=1e-6)
        done += 1
    assert done >= 40


def test_backward_invariants():
    rng = np.random.default_rng(12)
    for _ in range(50):
        n = int(rng.integers(2, 300))
        y = rng.standard_normal(n)
        lam = float(rng.uniform(0.05, 3))
        x = oracle.prox1d(y, lam)
        b, s = oracle.codes(x, lam)
        gy, ge, gl = oracle.bwd1d(b, s, np.ones(n))    # sum preservation => g = 1 passes, lam-grad 0
        np.testing.assert_allclose(gy, 1.0, atol=1e-14)
        assert abs(gl) < 1e-12
    # lam = 0: every edge a boundary, Jacobian = identity (reading O23)
    y = rng.standard_normal(20)
    b, s = oracle.codes(oracle.prox1d(y, 0.0), 0.0)
    assert b.all()
    g = rng.standard_normal(20)
    assert np.array_equal(oracle.bwd1d(b, s, g)[0], g)


def test_batch_matches_single():
    rng = np.random.default_rng(13)
    y = rng.standard_normal((37, 50))
    lam = rng.uniform(0.1, 1.0, size=37)
    x, brk, sgn = oracle.prox1d_batch(y, lam, nthreads=4)
    for r in range(37):
        assert np.array_equal(x[r], oracle.prox1d(y[r], lam[r]))
    g = rng.standard_normal((37, 50))
    gy, gl = oracle.bwd1d_batch(brk, sgn, g, nthreads=3)
    for r in range(37):
        a, _, t = oracle.bwd1d(brk[r], sgn[r], g[r])
        assert np.array_equal(gy[r], a) and gl[r] == t
