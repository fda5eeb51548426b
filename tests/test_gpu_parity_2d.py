"""GPU parity: 2D TV prox by Proximal Dykstra (Alg. 1) and its reverse
mode through the C ABI, vs the CPU oracle at the same K (reading O10)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2204_03643_b200 import workloads  # noqa: E402
from tests._util import TOL, codes_to_brk_sgn, rng_range, unpack_codes  # noqa: E402


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_03643_b200 import tvprox
    return tvprox


def plane_lams(lam, mode, N, C):
    if mode == "scalar":
        return np.full(N * C, float(lam))
    if mode == "channel":
        return np.tile(np.asarray(lam, np.float64), N)
    return np.asarray(lam, np.float64).reshape(N * C)


def saved_codes(saved, N, C, H, W, K):
    """Split the ABI's saved buffer into per-plane oracle segmentations [P][K][lines][n-1]."""
    P = N * C
    mwr = (W - 1 + 15) // 16 if W > 1 else 0
    mwc = (H - 1 + 15) // 16 if H > 1 else 0
    s = np.asarray(saved).astype(np.uint32)
    rs = K * P * H * mwr
    rows = s[:rs].reshape(K, P * H, max(mwr, 1) if mwr else 0) if mwr else np.zeros((K, P * H, 0), np.uint32)
    cols = s[rs:rs + K * P * W * mwc].reshape(K, P * W, mwc) if mwc else np.zeros((K, P * W, 0), np.uint32)
    rc = np.stack([unpack_codes(rows[k], W) for k in range(K)]).reshape(K, P, H, max(W - 1, 0))
    cc = np.stack([unpack_codes(cols[k], H) for k in range(K)]).reshape(K, P, W, max(H - 1, 0))
    rb, rsg = codes_to_brk_sgn(rc.transpose(1, 0, 2, 3))
    cb, csg = codes_to_brk_sgn(cc.transpose(1, 0, 2, 3))
    return (rb, rsg, cb, csg)


def run_case(tp, X, lam, mode, K, dtype=torch.float32, dkey="f32", grad_seed=1, check_bwd=True):
    N, C, H, W = X.shape
    Xt = torch.as_tensor(X, dtype=dtype, device="cuda")
    lt = lam if mode == "scalar" else torch.as_tensor(np.asarray(lam), dtype=dtype, device="cuda")
    Y, saved, it = tp.tv2d_fwd(Xt, lt, K, training=True, want_iters=True)
    torch.cuda.synchronize()
    Yg = Y.cpu().numpy().astype(np.float64)
    itn = it.cpu().numpy()
    assert np.all(itn < (1 << 20)), "some line did not converge: %s" % itn
    lamp = plane_lams(lam, mode, N, C)
    Xp = X.reshape(N * C, H, W).astype(np.float64)
    Yr, segs = oracle.prox2d_batch(Xp, lamp, K, nthreads=8)
    rng = rng_range(Xp)
    err = np.abs(Yg.reshape(N * C, H, W) - Yr).max()
    assert err <= TOL[dkey] * rng, "2D fwd err %.3e x range" % (err / rng)
    gsegs = saved_codes(saved.cpu().numpy(), N, C, H, W, K)
    # audit: mask disagreements vs the oracle's own segmentation (O13 ii/iii)
    dis = sum(int(((a != b)).sum()) for a, b in zip(gsegs, segs))
    total = sum(a.size for a in segs)
    if not check_bwd:
        return err / rng, dis, total
    G = np.random.default_rng(grad_seed).standard_normal(X.shape).astype(X.dtype)
    Gt = torch.as_tensor(G, dtype=dtype, device="cuda")
    mode_code = {"scalar": 0, "channel": 3, "plane": 4}[mode]
    GX, gl = tp.tv2d_bwd(Gt, saved, mode_code, K, want_lam=True)
    torch.cuda.synchronize()
    GXg = GX.cpu().numpy().astype(np.float64).reshape(N * C, H, W)
    GXr, glr = oracle.bwd2d_batch(gsegs, G.reshape(N * C, H, W).astype(np.float64), K, nthreads=8)
    grng = rng_range(G)
    gerr = np.abs(GXg - GXr).max()
    assert gerr <= TOL[dkey] * grng, "2D bwd err %.3e x range" % (gerr / grng)
    glg = gl.cpu().numpy().astype(np.float64)
    if mode == "scalar":
        ref = np.array([glr.sum()])
    elif mode == "channel":
        ref = glr.reshape(N, C).sum(0)
    else:
        ref = glr
    scale = np.abs(glr).sum() + 1.0
    assert np.abs(glg - ref).max() <= TOL[dkey] * scale
    return err / rng, dis, total


@pytest.mark.parametrize("H,W", [(1, 1), (1, 7), (7, 1), (2, 2), (3, 4), (5, 33), (33, 5), (16, 16),
                                 (56, 56), (64, 65), (100, 37), (224, 224), (129, 300), (20, 700),
                                 (700, 20), (9, 1024), (1024, 9)])
def test_shapes(tp, H, W):
    rng = np.random.default_rng(H * 1000 + W)
    X = rng.standard_normal((2, 2, H, W)).astype(np.float32)
    run_case(tp, X, [0.3, 0.9], "channel", 3, grad_seed=H + W)


@pytest.mark.parametrize("K", [1, 2, 4, 5])
def test_iters(tp, K):
    rng = np.random.default_rng(40 + K)
    X = np.maximum(rng.standard_normal((2, 3, 56, 56)), 0).astype(np.float32)
    run_case(tp, X, 0.5, "scalar", K)


def test_golden_3x4(tp):
    X = np.array([[0.3, 2.1, 1.4, 0.2], [3.2, 0.1, 1.3, 2.6], [1.1, 1.7, 4.2, 0.9]]).reshape(1, 1, 3, 4)
    for K in (1, 4):
        run_case(tp, X, 0.4, "scalar", K, dtype=torch.float64, dkey="f64")


def test_fp64_planes(tp):
    rng = np.random.default_rng(77)
    X = rng.standard_normal((1, 3, 40, 70))
    run_case(tp, X, rng.uniform(0.1, 1.0, 3), "plane", 4, dtype=torch.float64, dkey="f64")


def test_lambda_zero_identity(tp):
    X = np.random.default_rng(5).standard_normal((2, 2, 30, 40)).astype(np.float32)
    Xt = torch.as_tensor(X, device="cuda")
    Y, _, _ = tp.tv2d_fwd(Xt, 0.0, 4)
    torch.cuda.synchronize()
    assert np.array_equal(Y.cpu().numpy(), X)


def test_sum_preserved(tp):
    X = np.random.default_rng(6).standard_normal((1, 4, 64, 64))
    Y, _, _ = tp.tv2d_fwd(torch.as_tensor(X, device="cuda"), 0.8, 4)
    torch.cuda.synchronize()
    np.testing.assert_allclose(Y.cpu().numpy().sum((2, 3)), X.sum((2, 3)), atol=1e-9)


def test_autograd_2d(tp):
    rng = np.random.default_rng(8)
    X = torch.tensor(rng.standard_normal((1, 2, 12, 9)), device="cuda", requires_grad=True)
    lam = torch.tensor([0.3, 0.6], dtype=torch.float64, device="cuda", requires_grad=True)
    Y = tp.tv2d(X, lam, iters=3)
    G = torch.tensor(rng.standard_normal(Y.shape), device="cuda")
    (Y * G).sum().backward()
    Yr, segs = oracle.prox2d_batch(X.detach().cpu().numpy().reshape(2, 12, 9), np.array([0.3, 0.6]), 3)
    np.testing.assert_allclose(Y.detach().cpu().numpy().reshape(2, 12, 9), Yr, atol=1e-9)
    GXr, glr = oracle.bwd2d_batch(segs, G.cpu().numpy().reshape(2, 12, 9), 3)
    np.testing.assert_allclose(X.grad.cpu().numpy().reshape(2, 12, 9), GXr, atol=1e-9)
    np.testing.assert_allclose(lam.grad.cpu().numpy(), glr, atol=1e-9)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_config_shaped_small(tp, cfg):
    """The configs' generators and lambda recipes at reduced batch (every plane checked)."""
    if cfg == "C3":
        w = workloads.c3(N=2, C=64)
    elif cfg == "C4":
        w = workloads.c4(N=1, C=1)
    else:
        w = workloads.c5(N=2)
    lam = w.lam_scalar if w.lam_mode == "scalar" else w.lam.astype(np.float32)
    run_case(tp, w.X, lam, w.lam_mode, w.iters)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_config_full_size_sampled(tp, cfg):
    """BASELINE configs at full size in the bench's launch configuration; the oracle
    recomputes a seeded sample of planes one by one."""
    w = {"C3": workloads.c3, "C4": workloads.c4, "C5": workloads.c5}[cfg](with_grad=False)
    N, C, H, W = w.X.shape
    Xt = torch.as_tensor(w.X, device="cuda")
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    Y, saved, it = tp.tv2d_fwd(Xt, lam, w.iters, training=True, want_iters=True)
    torch.cuda.synchronize()
    assert np.all(it.cpu().numpy() < (1 << 20))
    picks = np.random.default_rng(3).choice(N * C, 4, replace=False)
    lamp = plane_lams(w.lam_scalar if w.lam_mode == "scalar" else w.lam, w.lam_mode, N, C)
    Yg = Y.cpu().numpy().reshape(N * C, H, W)
    Xp = w.X.reshape(N * C, H, W)
    rng = rng_range(Xp)
    for p in picks:
        Yr, _ = oracle.prox2d(Xp[p].astype(np.float64), lamp[p], w.iters)
        assert np.abs(Yg[p] - Yr).max() <= TOL["f32"] * rng


@pytest.mark.parametrize("H,W", [(56, 56), (224, 224), (37, 600)])
def test_inference_no_saved(tp, H, W):
    """training=False (no saved masks; warm starts from the workspace masks, coarse
    pre-pass / in-kernel coarse paths) matches the oracle like the training call."""
    rng = np.random.default_rng(77 + H + W)
    X = rng.standard_normal((2, 3, H, W)).astype(np.float32)
    lam = torch.as_tensor(np.array([0.2, 0.6, 1.4], np.float32), device="cuda")
    Y, saved, _ = tp.tv2d_fwd(torch.as_tensor(X, device="cuda"), lam, 4, training=False)
    assert saved is None
    Yr, _ = oracle.prox2d_batch(X.reshape(6, H, W).astype(np.float64),
                                np.tile([0.2, 0.6, 1.4], 2).astype(np.float64), 4, nthreads=8)
    err = np.abs(Y.cpu().numpy().reshape(6, H, W).astype(np.float64) - Yr).max()
    assert err <= TOL["f32"] * rng_range(X.astype(np.float64))


@pytest.mark.parametrize("H,W,K,mode,dt", [(56, 56, 4, "channel", "f32"), (33, 64, 3, "scalar", "f32"),
                                            (64, 40, 2, "plane", "f32"), (50, 61, 1, "channel", "f32"),
                                            (56, 56, 4, "channel", "f64"), (64, 64, 5, "scalar", "f32")])
def test_fused_plane_matches_staged_bitwise(tp, H, W, K, mode, dt):
    """f2: the on-chip plane kernel gives bitwise the staged passes' output, saved masks
    and iteration counts (same line solver, same lane geometry), and matches the oracle."""
    from paper_2204_03643_b200 import _lib
    lib = _lib.load()
    dtype = torch.float32 if dt == "f32" else torch.float64
    N, C = 3, 2
    rng = np.random.default_rng(H * 7 + W + K)
    X = np.maximum(rng.standard_normal((N, C, H, W)), 0).astype(np.float32 if dt == "f32" else np.float64)
    lam = {"scalar": 0.45, "channel": [0.1, 0.8], "plane": list(rng.uniform(0.05, 1.2, N * C))}[mode]
    Xt = torch.as_tensor(X, device="cuda")
    lt = lam if mode == "scalar" else torch.as_tensor(np.asarray(lam), dtype=dtype, device="cuda")
    outs = []
    prev = lib.tvp_set_fused2d(1)
    try:
        for fused in (1, 0):
            lib.tvp_set_fused2d(fused)
            Y, saved, it = tp.tv2d_fwd(Xt, lt, K, training=True, want_iters=True)
            torch.cuda.synchronize()
            outs.append((Y.cpu().numpy(), saved.cpu().numpy(), it.cpu().numpy()))
    finally:
        lib.tvp_set_fused2d(prev)
    (Yf, sf, itf), (Ys, ss, its) = outs
    # backward (f2 adjoint planes on chip vs the staged adjoint passes) on the same saved masks
    mode_id = {"scalar": 0, "channel": 3, "plane": 4}[mode]
    G = torch.as_tensor(rng.standard_normal(X.shape), dtype=dtype, device="cuda")
    sv = torch.as_tensor(sf, device="cuda")
    bouts = []
    try:
        for fused in (1, 0):
            lib.tvp_set_fused2d(fused)
            GX, gl = tp.tv2d_bwd(G, sv, mode_id, K, want_lam=True)
            torch.cuda.synchronize()
            bouts.append((GX.cpu().numpy(), gl.cpu().numpy()))
    finally:
        lib.tvp_set_fused2d(prev)
    assert np.array_equal(bouts[0][0].view(np.uint8), bouts[1][0].view(np.uint8)), "fused != staged grad_X"
    assert np.array_equal(bouts[0][1].view(np.uint8), bouts[1][1].view(np.uint8)), "fused != staged grad_lam"
    assert np.array_equal(Yf.view(np.uint8), Ys.view(np.uint8)), "fused != staged output"
    assert np.array_equal(sf, ss), "fused != staged saved masks"
    assert np.array_equal(itf, its)
    lamp = plane_lams(lam, mode, N, C)
    Yr, _ = oracle.prox2d_batch(X.reshape(N * C, H, W).astype(np.float64), lamp, K, nthreads=8)
    err = np.abs(Yf.reshape(N * C, H, W).astype(np.float64) - Yr).max()
    assert err <= TOL[dt] * rng_range(X.astype(np.float64))
