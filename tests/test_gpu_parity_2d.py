"""GPU parity: 2D TV prox by Proximal Dykstra (Alg. 1) and its reverse
mode through the C ABI, vs the CPU oracle at the same K (reading O10)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2204_03643_b200 import workloads  # noqa: E402
from tests._util import TOL, codes_to_brk_sgn, rng_range, taint_2d, unpack_codes  # noqa: E402


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


def audit_2d(gsegs, segs, jumps, rng, dkey):
    """Mask audit of a 2D forward (reading O13 (iii)): every edge of every pass where the
    GPU's saved mask disagrees with the oracle's own segmentation must be a near-degenerate
    edge, i.e. the oracle's output of that pass jumps there by at most 10 * tol * range."""
    grb, grs, gcb, gcs = gsegs
    orb, ors, ocb, ocs = segs
    rj, cj = jumps
    drow = (grb != orb) | (grs != ors)
    dcol = (gcb != ocb) | (gcs != ocs)
    bound = 10 * TOL[dkey] * rng
    if drow.any():
        assert np.abs(rj[drow]).max() <= bound, "row-mask disagreement at a non-degenerate edge: %.3e x range" % (
            np.abs(rj[drow]).max() / rng)
    if dcol.any():
        assert np.abs(cj[dcol]).max() <= bound, "column-mask disagreement at a non-degenerate edge: %.3e x range" % (
            np.abs(cj[dcol]).max() / rng)
    return int(drow.sum() + dcol.sum()), int(drow.size + dcol.size)


def run_case(tp, X, lam, mode, K, dtype=torch.float32, dkey="f32", grad_seed=1, check_bwd=True, opts=None,
             in_place=False):
    N, C, H, W = X.shape
    Xt = torch.as_tensor(X, dtype=dtype, device="cuda")
    lt = lam if mode == "scalar" else torch.as_tensor(np.asarray(lam), dtype=dtype, device="cuda")
    Xin = Xt.clone() if in_place else Xt
    Y, saved, it = tp.tv2d_fwd(Xin, lt, K, training=True, want_iters=True, opts=opts,
                               out=Xin if in_place else None)
    torch.cuda.synchronize()
    if in_place:
        assert Y.data_ptr() == Xin.data_ptr()
    Yg = Y.cpu().numpy().astype(np.float64)
    itn = it.cpu().numpy()
    assert np.all(itn < (1 << 20)), "some line did not converge: %s" % itn
    lamp = plane_lams(lam, mode, N, C)
    Xp = X.reshape(N * C, H, W).astype(np.float64)
    Yr, segs, jumps = oracle.prox2d_batch(Xp, lamp, K, nthreads=8, with_jumps=True)
    rng = rng_range(Xp)
    err = np.abs(Yg.reshape(N * C, H, W) - Yr).max()
    assert err <= TOL[dkey] * rng, "2D fwd err %.3e x range" % (err / rng)
    gsegs = saved_codes(saved.cpu().numpy(), N, C, H, W, K)
    # O13 (iii): disagreements with the oracle's own segmentation only at near-degenerate edges
    dis, total = audit_2d(gsegs, segs, jumps, rng, dkey)
    if not check_bwd:
        return err / rng, dis, total
    G = np.random.default_rng(grad_seed).standard_normal(X.shape).astype(X.dtype)
    Gt = torch.as_tensor(G, dtype=dtype, device="cuda")
    mode_code = {"scalar": 0, "channel": 3, "plane": 4}[mode]
    Gin = Gt.clone() if in_place else Gt
    GX, gl = tp.tv2d_bwd(Gin, saved, mode_code, K, want_lam=True, opts=opts, out=Gin if in_place else None)
    torch.cuda.synchronize()
    GXg = GX.cpu().numpy().astype(np.float64).reshape(N * C, H, W)
    G64 = G.reshape(N * C, H, W).astype(np.float64)
    # O13 (i): the oracle's reverse mode on the GPU's own masks, everywhere
    GXr, glr = oracle.bwd2d_batch(gsegs, G64, K, nthreads=8)
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
    # O13 (ii): the oracle's reverse mode on ITS OWN masks must match wherever no mask
    # disagreement can reach (taint propagated through the 2K adjoint passes)
    GXo, glo = oracle.bwd2d_batch(segs, G64, K, nthreads=8)
    tainted = taint_2d(gsegs, segs, H, W, K)
    if (~tainted).any():
        oerr = np.abs(GXg - GXo)[~tainted].max()
        assert oerr <= TOL[dkey] * grng, "2D bwd vs oracle-own masks %.3e x range off the tainted set" % (oerr / grng)
    if mode == "plane":
        clean = ~tainted.reshape(N * C, -1).any(1)
        if clean.any():
            assert np.abs(glg[clean] - glo[clean]).max() <= TOL[dkey] * scale
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


def plane_segs(saved, N, C, H, W, K, planes):
    """Oracle-layout segmentations (rbrk, rsgn, cbrk, csgn) of selected planes, read straight
    out of the ABI's saved buffer (K row-mask sets [P][H][mwr], then K column-mask sets)."""
    P = N * C
    mwr = (W - 1 + 15) // 16 if W > 1 else 0
    mwc = (H - 1 + 15) // 16 if H > 1 else 0
    s = np.asarray(saved).astype(np.uint32)
    rows = s[:K * P * H * mwr].reshape(K, P, H, mwr)[:, planes]
    cols = s[K * P * H * mwr:K * P * H * mwr + K * P * W * mwc].reshape(K, P, W, mwc)[:, planes]
    S = len(planes)
    rc = np.stack([unpack_codes(rows[k].reshape(S * H, mwr), W) for k in range(K)]).reshape(K, S, H, max(W - 1, 0))
    cc = np.stack([unpack_codes(cols[k].reshape(S * W, mwc), H) for k in range(K)]).reshape(K, S, W, max(H - 1, 0))
    rb, rsg = codes_to_brk_sgn(rc.transpose(1, 0, 2, 3))
    cb, csg = codes_to_brk_sgn(cc.transpose(1, 0, 2, 3))
    return (rb, rsg, cb, csg)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_config_full_size_sampled(tp, cfg):
    """BASELINE configs at full size in the bench's launch configuration (forward with saved
    masks, backward with the per-channel / scalar lambda gradient); the oracle recomputes 32
    seeded planes one by one: forward parity and mask audit (O13 iii), backward on the GPU's
    masks (O13 i) and on the oracle's own masks off the tainted set (O13 ii)."""
    w = {"C3": workloads.c3, "C4": workloads.c4, "C5": workloads.c5}[cfg](with_grad=True)
    N, C, H, W = w.X.shape
    K = w.iters
    Xt = torch.as_tensor(w.X, device="cuda")
    lam = w.lam_scalar if w.lam_mode == "scalar" else torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    Y, saved, it = tp.tv2d_fwd(Xt, lam, K, training=True, want_iters=True)
    mode_code = {"scalar": 0, "channel": 3, "plane": 4}[w.lam_mode]
    GX, gl = tp.tv2d_bwd(torch.as_tensor(w.grad, device="cuda"), saved, mode_code, K, want_lam=True)
    torch.cuda.synchronize()
    assert np.all(it.cpu().numpy() < (1 << 20))
    assert torch.isfinite(GX).all() and torch.isfinite(gl).all()
    picks = np.sort(np.random.default_rng(3).choice(N * C, 32, replace=False))
    lamp = plane_lams(w.lam_scalar if w.lam_mode == "scalar" else w.lam, w.lam_mode, N, C)[picks]
    Xp = w.X.reshape(N * C, H, W)[picks].astype(np.float64)
    Yg = Y.cpu().numpy().reshape(N * C, H, W)[picks].astype(np.float64)
    rng = rng_range(w.X)
    Yr, segs, jumps = oracle.prox2d_batch(Xp, lamp, K, nthreads=8, with_jumps=True)
    assert np.abs(Yg - Yr).max() <= TOL["f32"] * rng
    gsegs = plane_segs(saved.cpu().numpy(), N, C, H, W, K, picks)
    dis, total = audit_2d(gsegs, segs, jumps, rng, "f32")
    G64 = w.grad.reshape(N * C, H, W)[picks].astype(np.float64)
    GXg = GX.cpu().numpy().reshape(N * C, H, W)[picks].astype(np.float64)
    grng = rng_range(w.grad)
    GXr, _ = oracle.bwd2d_batch(gsegs, G64, K, nthreads=8)
    assert np.abs(GXg - GXr).max() <= TOL["f32"] * grng
    GXo, _ = oracle.bwd2d_batch(segs, G64, K, nthreads=8)
    tainted = taint_2d(gsegs, segs, H, W, K)
    if (~tainted).any():
        assert np.abs(GXg - GXo)[~tainted].max() <= TOL["f32"] * grng
    print("%s: %d mask disagreements in %d edge-passes, %.1f%% of sampled pixels tainted"
          % (cfg, dis, total, 100.0 * tainted.mean()))


def test_huge_lambda_global_mean(tp):
    """lam above the row lam_max and then the column lam_max of the row-mean image: the 2D
    prox of Alg. 1 is the plane's global mean after K = 1 and stays there (SURVEY 8(c) pin)."""
    rng = np.random.default_rng(11)
    X = rng.standard_normal((2, 3, 40, 70)).astype(np.float32)
    for K in (1, 4):
        Y, _, _ = tp.tv2d_fwd(torch.as_tensor(X, device="cuda"), 1.0e4, K)
        torch.cuda.synchronize()
        Yn = Y.cpu().numpy().astype(np.float64)
        mean = X.astype(np.float64).mean((2, 3), keepdims=True)
        assert np.abs(Yn - mean).max() <= TOL["f32"] * rng_range(X)
    run_case(tp, X, 1.0e4, "scalar", 4)
    run_case(tp, X[:, :, :56, :56].copy(), [1e4, 5e3, 2e4], "channel", 3)      # fused plane path


@pytest.mark.parametrize("H,W", [(56, 56), (100, 37), (224, 224)])
def test_in_place(tp, H, W):
    """Y == X and grad_X == grad_Y (include/tvprox.h allows both): same results as out of place."""
    rng = np.random.default_rng(H + 3 * W)
    X = np.maximum(rng.standard_normal((2, 3, H, W)), 0).astype(np.float32)
    run_case(tp, X, [0.2, 0.5, 1.1], "channel", 4, in_place=True)


@pytest.mark.parametrize("H,W,fused", [(56, 56, -1), (56, 56, 0), (224, 224, 0), (224, 224, 1), (40, 300, 0)])
def test_nonfinite_pixel_isolated_to_its_plane(tp, H, W, fused):
    """A NaN pixel poisons its own plane (its row, then the columns that row reaches) and
    flags the passes as not converged; every other plane is exact (O21 per line)."""
    rng = np.random.default_rng(H * 5 + W)
    X = np.maximum(rng.standard_normal((2, 2, H, W)), 0).astype(np.float32)
    X[1, 0, H // 3, W // 2] = np.nan
    lam = np.array([0.3, 0.9], np.float32)
    Y, saved, li = tp.tv2d_fwd(torch.as_tensor(X, device="cuda"), torch.as_tensor(lam, device="cuda"), 4,
                               want_iters=True, opts=tp.make_options(fused2d=fused))
    Y = Y.cpu().numpy().reshape(4, H, W)
    assert np.isnan(Y[2]).any()
    assert np.all(li.cpu().numpy()[0] >= (1 << 20))          # row pass 1 saw a non-finite line
    good = [0, 1, 3]
    Yr, _ = oracle.prox2d_batch(X.reshape(4, H, W)[good].astype(np.float64), np.tile(lam, 2)[good].astype(np.float64),
                                4, nthreads=8)
    assert np.all(np.isfinite(Y[good]))
    assert np.abs(Y[good].astype(np.float64) - Yr).max() <= TOL["f32"] * rng_range(X.reshape(4, H, W)[good])


@pytest.mark.parametrize("H,W", [(1024, 9), (9, 1024), (600, 20), (20, 600)])
def test_fp64_long_lines(tp, H, W):
    """fp64 rows and columns of 513..1024 samples (E = 32 geometry; columns on 4-warp tiles
    that fit the 227 KB shared-memory limit)."""
    rng = np.random.default_rng(H * 7 + W)
    X = rng.standard_normal((1, 2, H, W))
    run_case(tp, X, [0.4, 1.3], "channel", 2, dtype=torch.float64, dkey="f64")


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
                                            (56, 56, 4, "channel", "f64"), (64, 64, 5, "scalar", "f32"),
                                            # thread-block-cluster f2 (65..224 per side, fp32)
                                            (224, 224, 4, "channel", "f32"), (150, 200, 3, "scalar", "f32"),
                                            (224, 129, 2, "plane", "f32"), (128, 128, 4, "channel", "f32"),
                                            (70, 100, 1, "scalar", "f32"), (97, 65, 5, "plane", "f32")])
def test_fused_plane_matches_staged_bitwise(tp, H, W, K, mode, dt):
    """f2: the on-chip plane kernel gives bitwise the staged passes' output, saved masks
    and iteration counts (same line solver, same lane geometry), and matches the oracle."""
    dtype = torch.float32 if dt == "f32" else torch.float64
    N, C = 3, 2
    rng = np.random.default_rng(H * 7 + W + K)
    X = np.maximum(rng.standard_normal((N, C, H, W)), 0).astype(np.float32 if dt == "f32" else np.float64)
    lam = {"scalar": 0.45, "channel": [0.1, 0.8], "plane": list(rng.uniform(0.05, 1.2, N * C))}[mode]
    Xt = torch.as_tensor(X, device="cuda")
    lt = lam if mode == "scalar" else torch.as_tensor(np.asarray(lam), dtype=dtype, device="cuda")
    outs = []
    for fused in (1, 0):                      # per-call switch (tvp_options_t.fused2d)
        Y, saved, it = tp.tv2d_fwd(Xt, lt, K, training=True, want_iters=True, opts=tp.make_options(fused2d=fused))
        torch.cuda.synchronize()
        outs.append((Y.cpu().numpy(), saved.cpu().numpy(), it.cpu().numpy()))
    (Yf, sf, itf), (Ys, ss, its) = outs
    # backward (f2 adjoint planes on chip vs the staged adjoint passes) on the same saved masks
    mode_id = {"scalar": 0, "channel": 3, "plane": 4}[mode]
    G = torch.as_tensor(rng.standard_normal(X.shape), dtype=dtype, device="cuda")
    sv = torch.as_tensor(sf, device="cuda")
    bouts = []
    for fused in (1, 0):
        GX, gl = tp.tv2d_bwd(G, sv, mode_id, K, want_lam=True, opts=tp.make_options(fused2d=fused))
        torch.cuda.synchronize()
        bouts.append((GX.cpu().numpy(), gl.cpu().numpy()))
    assert np.array_equal(bouts[0][0].view(np.uint8), bouts[1][0].view(np.uint8)), "fused != staged grad_X"
    assert np.array_equal(bouts[0][1].view(np.uint8), bouts[1][1].view(np.uint8)), "fused != staged grad_lam"
    assert np.array_equal(Yf.view(np.uint8), Ys.view(np.uint8)), "fused != staged output"
    assert np.array_equal(sf, ss), "fused != staged saved masks"
    assert np.array_equal(itf, its)
    lamp = plane_lams(lam, mode, N, C)
    Yr, _ = oracle.prox2d_batch(X.reshape(N * C, H, W).astype(np.float64), lamp, K, nthreads=8)
    err = np.abs(Yf.reshape(N * C, H, W).astype(np.float64) - Yr).max()
    assert err <= TOL[dt] * rng_range(X.astype(np.float64))
