"""Pins for the 2D oracle (Algorithm 1, and its reverse mode).

Independent checks: SPEC's worked example, closed forms (constant-column
separability, huge-lam global mean), the paper's lam = 0 identity, sum
preservation, convergence of Algorithm 1 (K -> inf) to the exact 2D prox of
Eq. 2 computed by an independent projected-gradient dual solver, and central
finite differences of the K-unrolled map for the backward.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_spec_example():
    # [[0,2],[0,2]], lam=.5, K=4 -> [[.5,1.5],[.5,1.5]]
    Y, _ = oracle.prox2d(np.array([[0.0, 2.0], [0.0, 2.0]]), 0.5, 4)
    np.testing.assert_allclose(Y, [[0.5, 1.5], [0.5, 1.5]], atol=1e-15)


def test_lambda_zero_identity():
    rng = np.random.default_rng(20)
    X = rng.standard_normal((7, 9))
    for K in (1, 3):
        Y, _ = oracle.prox2d(X, 0.0, K)
        assert np.array_equal(Y, X)
        GX, gl = oracle.bwd2d(oracle.prox2d(X, 0.0, K)[1], X * 0 + 1.5, K)
        np.testing.assert_allclose(GX, 1.5, atol=1e-15)
        assert gl == 0.0


def test_constant_columns_reduce_to_rows():
    # all rows equal => the row prox output has constant columns, the column pass is the
    # identity and the Dykstra state is a fixed point: Y = row prox at every K.
    rng = np.random.default_rng(21)
    for K in (1, 2, 4):
        r = rng.standard_normal(11)
        X = np.tile(r, (6, 1))
        Y, _ = oracle.prox2d(X, 0.4, K)
        exp = np.tile(oracle.prox1d(r, 0.4), (6, 1))
        np.testing.assert_allclose(Y, exp, atol=1e-13)


def test_huge_lambda_global_mean():
    rng = np.random.default_rng(22)
    X = rng.standard_normal((5, 8))
    Y, _ = oracle.prox2d(X, 1e3, 1)
    np.testing.assert_allclose(Y, np.full_like(X, X.mean()), atol=1e-12)


def test_sum_preserved_every_K():
    rng = np.random.default_rng(23)
    X = rng.standard_normal((9, 13))
    for K in range(1, 6):
        Y, _ = oracle.prox2d(X, 0.6, K)
        assert abs(Y.sum() - X.sum()) < 1e-11


def test_golden_3x4():
    with open(os.path.join(GOLDEN, "tv2d.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        X = np.array(case["X"])
        Y, segs = oracle.prox2d(X, case["lam"], case["K"])
        np.testing.assert_allclose(Y, np.array(case["Y"]), atol=1e-11, err_msg=case["cite"])
        GX, gl = oracle.bwd2d(segs, np.array(case["G"]), case["K"])
        np.testing.assert_allclose(GX, np.array(case["grad_X"]), atol=1e-11, err_msg=case["cite"])
        assert abs(gl - case["grad_lam"]) < 1e-11


def pgd_dual_2d(X, lam, iters=60000):
    """Exact anisotropic 2D prox (Eq. 2) by projected gradient on its dual:
    Y = X - Dh^T uh - Dv^T uv, |u| <= lam, step 1/8 (||[Dh;Dv]||^2 <= 8).  Independent."""
    H, W = X.shape
    uh = np.zeros((H, W - 1))
    uv = np.zeros((H - 1, W))
    for _ in range(iters):
        Y = X.copy()
        Y[:, :-1] += uh
        Y[:, 1:] -= uh
        Y[:-1, :] += uv
        Y[1:, :] -= uv
        uh = np.clip(uh + 0.125 * np.diff(Y, axis=1), -lam, lam)
        uv = np.clip(uv + 0.125 * np.diff(Y, axis=0), -lam, lam)
    Y = X.copy()
    Y[:, :-1] += uh
    Y[:, 1:] -= uh
    Y[:-1, :] += uv
    Y[1:, :] -= uv
    return Y


def test_dykstra_converges_to_exact_2d_prox():
    # Proximal Dykstra (Alg. 1) converges to Prox_TV^2D of Eq. 2 as K grows.
    rng = np.random.default_rng(24)
    X = rng.standard_normal((6, 6))
    ref = pgd_dual_2d(X, 0.3)
    Y, _ = oracle.prox2d(X, 0.3, 400)
    np.testing.assert_allclose(Y, ref, atol=2e-5)


def _fd_stable(X, lam, K, segs, dirs, h):
    for D in dirs:
        for s in (h, -h):
            _, sg = oracle.prox2d(X + s * D, lam, K)
            if any(not np.array_equal(a, b) for a, b in zip(sg, segs)):
                return False
    return True


@pytest.mark.parametrize("K", [1, 2, 3])
def test_backward_finite_differences(K):
    rng = np.random.default_rng(30 + K)
    h = 1e-6
    done = 0
    for trial in range(20):
        H, W = 6, 6
        X = rng.standard_normal((H, W))
        lam = 0.7
        Y, segs = oracle.prox2d(X, lam, K)
        G = rng.standard_normal((H, W))
        GX, gl = oracle.bwd2d(segs, G, K)
        dirs = [np.eye(H * W)[i].reshape(H, W) for i in range(H * W)]
        if not _fd_stable(X, lam, K, segs, dirs, h):
            continue
        fd = np.array([(np.sum(G * oracle.prox2d(X + h * D, lam, K)[0]) -
                        np.sum(G * oracle.prox2d(X - h * D, lam, K)[0])) / (2 * h) for D in dirs])
        np.testing.assert_allclose(GX.ravel(), fd, atol=2e-6)
        _, s1 = oracle.prox2d(X, lam + h, K)
        _, s2 = oracle.prox2d(X, lam - h, K)
        if all(np.array_equal(a, b) for a, b in zip(s1, segs)) and all(np.array_equal(a, b) for a, b in zip(s2, segs)):
            fdl = (np.sum(G * oracle.prox2d(X, lam + h, K)[0]) - np.sum(G * oracle.prox2d(X, lam - h, K)[0])) / (2 * h)
            assert abs(gl - fdl) < 2e-6
        done += 1
        if done >= 3:
            break
    assert done >= 1


def test_backward_ones_invariant():
    # sum(Y) = sum(X) at every K => G = 1 gives grad_X = 1 and grad_lam = 0
    rng = np.random.default_rng(40)
    X = rng.standard_normal((10, 7))
    for K in (1, 4):
        _, segs = oracle.prox2d(X, 0.5, K)
        GX, gl = oracle.bwd2d(segs, np.ones_like(X), K)
        np.testing.assert_allclose(GX, 1.0, atol=1e-13)
        assert abs(gl) < 1e-12


def test_batch_matches_single():
    rng = np.random.default_rng(41)
    X = rng.standard_normal((5, 9, 8))
    lam = np.array([0.1, 0.5, 0.0, 1.0, 3.0])
    Y, segs = oracle.prox2d_batch(X, lam, 3, nthreads=3)
    G = rng.standard_normal(X.shape)
    GX, gl = oracle.bwd2d_batch(segs, G, 3, nthreads=2)
    for p in range(5):
        y1, s1 = oracle.prox2d(X[p], lam[p], 3)
        assert np.array_equal(Y[p], y1)
        for a, b in zip(s1, segs):
            assert np.array_equal(a, b[p])
        g1, l1 = oracle.bwd2d(s1, G[p], 3)
        assert np.array_equal(GX[p], g1) and gl[p] == l1
