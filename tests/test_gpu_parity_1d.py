"""GPU parity: batched 1D TV prox (libtvprox.so through the C ABI) vs the CPU oracle.

Bar (north_star): forward max-abs error <= tol * range(y), tol 1e-4 (fp32) / 1e-9
(fp64); backward mask-aware (O13): the oracle's VJP evaluated on the
GPU's own segmentation must match element by element, and every edge where
the GPU segmentation differs from the oracle's must be a near-degenerate edge.
"""
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


def run_gpu(tp, y, lam, dtype):
    yt = torch.as_tensor(y, dtype=dtype, device="cuda")
    if isinstance(lam, np.ndarray):
        lam = torch.as_tensor(lam, dtype=dtype, device="cuda")
    x, mask, it = tp.tv1d_fwd(yt, lam, need_mask=True, want_iters=True)
    torch.cuda.synchronize()
    return x.cpu().numpy(), mask.cpu().numpy(), it.cpu().numpy()


def check_forward(y, lam, x_gpu, mask, iters, dkey, per_edge=False):
    b, n = y.shape
    y64 = y.astype(np.float64)
    if np.ndim(lam) == 0:
        lamr = np.full(b, float(lam))
        x_ref, brk, sgn = oracle.prox1d_batch(y64, lamr, nthreads=8)
    elif per_edge:
        x_ref, brk, sgn = oracle.prox1d_batch(y64, np.asarray(lam, np.float64), per_edge=True, nthreads=8)
    else:
        x_ref, brk, sgn = oracle.prox1d_batch(y64, np.asarray(lam, np.float64), nthreads=8)
    rng = max(rng_range(y64), 1e-30)
    err = np.abs(x_gpu.astype(np.float64) - x_ref)
    assert np.all(iters >= 0), "rows not converged: %s" % np.unique(iters[iters < 0])
    assert err.max() <= TOL[dkey] * rng, "max err %.3e x range" % (err.max() / rng)
    # mask audit: disagreements only at near-degenerate edges (O13 iii)
    codes = unpack_codes(mask, n)
    gb, gs = codes_to_brk_sgn(codes)
    dis = (gb != brk) | (gs != sgn)
    if dis.any():
        dxr = np.abs(np.diff(x_ref, axis=1))
        assert np.all(dxr[dis] <= 10 * TOL[dkey] * rng), "mask disagreement at a non-degenerate edge"
    return x_ref, codes, dis.sum()


@pytest.mark.parametrize("n", [1, 2, 3, 5, 16, 17, 31, 32, 33, 56, 63, 64, 65, 100, 128, 129, 200, 224,
                               225, 255, 256, 257, 400, 512, 513, 777, 1000, 1023, 1024])
@pytest.mark.parametrize("kind", ["normal", "step"])
def test_forward_sizes_fp32(tp, n, kind):
    y = workloads.random_rows(7000 + n, 37, n, kind, np.float32)
    lam = np.random.default_rng(n).uniform(0.05, 1.5, 37)
    x, mask, it = run_gpu(tp, y, lam.astype(np.float32), torch.float32)
    check_forward(y, lam.astype(np.float32).astype(np.float64), x, mask, it, "f32")


@pytest.mark.parametrize("n", [17, 56, 100, 224, 300, 512, 1024, 3000])
@pytest.mark.parametrize("dt", ["f32", "f64"])
def test_forward_degenerate_ties(tp, n, dt):
    """Integer-valued rows with integer / half-integer lambda: exact ties everywhere (|uhat|
    equal to lambda on free edges, zero-height jumps, equal segment means) -- the inputs
    where the rounding-level stall rules decide termination (O8).
    Every row's output meets the parity bar; a few rows may end at max_iters (row_iters
    -1, output x(u) of the last dual, known limitation), at most 1 in 16."""
    npdt, tdt = (np.float32, torch.float32) if dt == "f32" else (np.float64, torch.float64)
    y = workloads.random_rows(7400 + n, 64, n, "int", npdt)
    lam = np.random.default_rng(n + 1).integers(1, 7, 64) * 0.5
    x, mask, it = run_gpu(tp, y, lam.astype(npdt), tdt)
    x_ref, _, _ = oracle.prox1d_batch(y.astype(np.float64), lam, nthreads=8)
    rng = max(rng_range(y.astype(np.float64)), 1e-30)
    assert np.abs(x.astype(np.float64) - x_ref).max() <= TOL[dt] * rng
    assert np.all((it >= 0) | (it == -1))
    assert (it == -1).sum() <= len(it) // 16
    ok = it >= 0
    if ok.any():
        check_forward(y[ok], lam[ok], x[ok], mask[ok], it[ok], dt)


@pytest.mark.parametrize("n", [1, 2, 7, 33, 64, 65, 224, 512, 1024])
def test_forward_sizes_fp64(tp, n):
    y = workloads.random_rows(8000 + n, 21, n, "normal", np.float64)
    lam = np.random.default_rng(n).uniform(0.05, 1.5, 21)
    x, mask, it = run_gpu(tp, y, lam, torch.float64)
    check_forward(y, lam, x, mask, it, "f64")


def _bwd_compare(tp, y, lam, mode_lam, dtype, dkey, seed):
    b, n = y.shape
    x, mask, it = run_gpu(tp, y, lam, dtype)
    per_edge = isinstance(lam, np.ndarray) and lam.ndim == 2
    lam64 = np.asarray(lam, np.float64) if isinstance(lam, np.ndarray) else lam
    x_ref, codes, _ = check_forward(y, lam64, x, mask, it, dkey, per_edge=per_edge)
    g = np.random.default_rng(seed).standard_normal((b, n)).astype(np.float32 if dkey == "f32" else np.float64)
    gt = torch.as_tensor(g, device="cuda")
    mt = torch.as_tensor(mask, device="cuda")
    gy, gl = tp.tv1d_bwd(gt, mt, mode_lam, want_lam=True)
    torch.cuda.synchronize()
    gy = gy.cpu().numpy().astype(np.float64)
    gl = gl.cpu().numpy().astype(np.float64)
    brk, sgn = codes_to_brk_sgn(codes)
    gy_ref, gl_ref = oracle.bwd1d_batch(brk, sgn, g.astype(np.float64), per_edge=per_edge, nthreads=8)
    grng = rng_range(g)
    assert np.abs(gy - gy_ref).max() <= TOL[dkey] * grng
    if mode_lam == 0:   # scalar
        ref = gl_ref.sum()
        scale = np.abs(gl_ref).sum() + 1.0
        assert abs(gl[0] - ref) <= TOL[dkey] * scale
    elif per_edge:
        assert np.abs(gl - gl_ref).max() <= TOL[dkey] * (np.abs(gl_ref).max() + 1.0)
    else:
        assert np.abs(gl - gl_ref).max() <= TOL[dkey] * (np.abs(gl_ref).max() + 1.0)


@pytest.mark.parametrize("n", [2, 33, 64, 200, 512, 1024])
def test_backward_per_row(tp, n):
    y = workloads.random_rows(9000 + n, 40, n, "step", np.float32)
    lam = np.random.default_rng(n + 1).uniform(0.05, 1.0, 40).astype(np.float32)
    _bwd_compare(tp, y, lam, 1, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [2, 33, 300, 1024])
def test_backward_scalar(tp, n):
    y = workloads.random_rows(9100 + n, 40, n, "normal", np.float32)
    _bwd_compare(tp, y, 0.7, 0, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [3, 40, 129, 1024])
def test_per_edge_lambda(tp, n):
    rng = np.random.default_rng(9200 + n)
    y = rng.standard_normal((30, n)).astype(np.float32)
    lam = rng.uniform(0.0, 1.2, (30, n - 1)).astype(np.float32)
    lam[rng.random(lam.shape) < 0.1] = 0.0
    _bwd_compare(tp, y, lam, 2, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [1025, 1500, 2048, 2049, 3333, 4096, 6000, 8192])
@pytest.mark.parametrize("kind", ["normal", "step"])
def test_forward_long_rows_fp32(tp, n, kind):
    """f4 (long 1D signals): one CTA of 4-16 warps per row, ragged tails included."""
    y = workloads.random_rows(9400 + n, 9, n, kind, np.float32)
    lam = np.random.default_rng(n + 5).uniform(0.05, 2.0, 9)
    x, mask, it = run_gpu(tp, y, lam.astype(np.float32), torch.float32)
    check_forward(y, lam.astype(np.float32).astype(np.float64), x, mask, it, "f32")


@pytest.mark.parametrize("n", [1025, 2048, 3000, 4096])
def test_forward_long_rows_fp64(tp, n):
    y = workloads.random_rows(9500 + n, 6, n, "step", np.float64)
    lam = np.random.default_rng(n + 6).uniform(0.05, 2.0, 6)
    x, mask, it = run_gpu(tp, y, lam, torch.float64)
    check_forward(y, lam, x, mask, it, "f64")


@pytest.mark.parametrize("n", [1500, 4096, 8192])
def test_backward_long_rows(tp, n):
    y = workloads.random_rows(9600 + n, 8, n, "step", np.float32)
    lam = np.random.default_rng(n + 7).uniform(0.05, 1.0, 8).astype(np.float32)
    _bwd_compare(tp, y, lam, 1, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [2000, 8192])
def test_per_edge_lambda_long_rows(tp, n):
    rng = np.random.default_rng(9700 + n)
    y = rng.standard_normal((6, n)).astype(np.float32)
    lam = rng.uniform(0.0, 1.2, (6, n - 1)).astype(np.float32)
    lam[rng.random(lam.shape) < 0.1] = 0.0
    _bwd_compare(tp, y, lam, 2, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [100, 224, 300, 700, 1024, 3000])
def test_forward_inference_no_mask(tp, n):
    """need_mask=False (inference): the in-kernel coarse solve replaces the pre-pass."""
    y = workloads.random_rows(9800 + n, 24, n, "step", np.float32)
    lam = np.random.default_rng(n + 8).uniform(0.05, 1.5, 24).astype(np.float32)
    yt = torch.as_tensor(y, device="cuda")
    x, mask, it = tp.tv1d_fwd(yt, torch.as_tensor(lam, device="cuda"), need_mask=False, want_iters=True)
    assert mask is None
    x = x.cpu().numpy().astype(np.float64)
    assert np.all(it.cpu().numpy() >= 0)
    x_ref, _, _ = oracle.prox1d_batch(y.astype(np.float64), lam.astype(np.float64), nthreads=8)
    assert np.abs(x - x_ref).max() <= TOL["f32"] * rng_range(y.astype(np.float64))


@pytest.mark.parametrize("n,nrows", [(8193, 5), (12000, 4), (16384, 4), (30000, 3), (48000, 3), (65536, 2)])
def test_forward_cluster_rows_fp32(tp, n, nrows):
    """f4 past one CTA: a thread-block cluster of 2-16 CTAs holds the row in registers."""
    y = workloads.random_rows(9900 + n, nrows, n, "step", np.float32)
    lam = np.random.default_rng(n + 9).uniform(0.05, 2.0, nrows).astype(np.float32)
    x, mask, it = run_gpu(tp, y, lam, torch.float32)
    check_forward(y, lam.astype(np.float64), x, mask, it, "f32")


@pytest.mark.parametrize("n", [16384, 32768, 65536])
def test_forward_cluster_rows_noisy_fp32(tp, n):
    """The bench's f4 workload (C2's generator at length n, sigma 0.1 / 0.5 alternating,
    lambda scaled by sqrt(n/1024)): every row converges (cycles of period <= 4 accepted
    as rounding-level stalls, O7) and matches the oracle."""
    w = workloads.long_rows(n, batch=8)
    x, mask, it = run_gpu(tp, w.y, w.lam.astype(np.float32), torch.float32)
    check_forward(w.y, w.lam.astype(np.float32).astype(np.float64), x, mask, it, "f32")


@pytest.mark.parametrize("n", [4097, 10000, 32768, 65536])
def test_forward_cluster_rows_fp64(tp, n):
    y = workloads.random_rows(9950 + n, 2, n, "normal", np.float64)
    lam = np.random.default_rng(n + 10).uniform(0.05, 2.0, 2)
    x, mask, it = run_gpu(tp, y, lam, torch.float64)
    check_forward(y, lam, x, mask, it, "f64")


@pytest.mark.parametrize("n", [16384, 48000, 65536])
def test_backward_cluster_rows(tp, n):
    y = workloads.random_rows(9960 + n, 3, n, "step", np.float32)
    lam = np.random.default_rng(n + 11).uniform(0.05, 1.0, 3).astype(np.float32)
    _bwd_compare(tp, y, lam, 1, torch.float32, "f32", n)


@pytest.mark.parametrize("n", [20000])
def test_per_edge_lambda_cluster_rows(tp, n):
    rng = np.random.default_rng(9970 + n)
    y = rng.standard_normal((2, n)).astype(np.float32)
    lam = rng.uniform(0.0, 1.2, (2, n - 1)).astype(np.float32)
    lam[rng.random(lam.shape) < 0.1] = 0.0
    _bwd_compare(tp, y, lam, 2, torch.float32, "f32", n)


def test_long_row_limit(tp):
    from paper_2204_03643_b200 import _lib
    lib = _lib.load()
    assert lib.tvp_max_line_1d(_lib.TVP_F32) == 65536 and lib.tvp_max_line_1d(_lib.TVP_F64) == 65536
    y = torch.zeros((2, 65537), device="cuda")
    with pytest.raises(Exception):
        tp.tv1d_fwd(y, 0.5)


def test_c1_fp64_full(tp):
    w = workloads.c1()
    _bwd_compare(tp, w.y, w.lam_scalar, 0, torch.float64, "f64", 11)
    _bwd_compare(tp, w.y, w.lam.astype(np.float64), 1, torch.float64, "f64", 12)


def test_lambda_zero_identity_bitwise(tp):
    y = workloads.random_rows(9300, 17, 300, "normal", np.float32)
    x, mask, it = run_gpu(tp, y, 0.0, torch.float32)
    assert np.array_equal(x, y)
    codes = unpack_codes(mask, 300)
    assert np.all(codes != 0)          # every edge is a boundary at lam = 0 (O23)
    x, _, _ = run_gpu(tp, y, np.zeros(17, np.float32), torch.float32)
    assert np.array_equal(x, y)


def test_constant_rows_and_lambda_max(tp):
    y = workloads.random_rows(9400, 16, 500, "const", np.float32)
    x, mask, it = run_gpu(tp, y, 0.5, torch.float32)
    assert np.abs(x - y).max() <= 1e-6 * (np.abs(y).max() + 1)
    y = workloads.random_rows(9401, 16, 500, "normal", np.float64)
    lmax = np.abs(np.cumsum(y - y.mean(1, keepdims=True), axis=1)[:, :-1]).max(1)
    x, mask, it = run_gpu(tp, y, lmax * 1.01, torch.float64)
    np.testing.assert_allclose(x, np.repeat(y.mean(1, keepdims=True), 500, 1), atol=1e-12)
    assert np.all(unpack_codes(mask, 500) == 0)


def test_nonfinite_row_flagged(tp):
    y = workloads.random_rows(9500, 8, 100, "normal", np.float32)
    y[3, 17] = np.nan
    x, mask, it = run_gpu(tp, y, 0.5, torch.float32)
    assert it[3] == -2 and np.all(np.isnan(x[3]))
    others = [i for i in range(8) if i != 3]
    check_forward(y[others], 0.5, x[others], mask[others], it[others], "f32")


@pytest.mark.parametrize("n", [3000, 20000])
def test_long_rows_edge_cases(tp, n):
    """One-CTA and cluster long rows: lambda = 0 is a bitwise copy, a NaN row is flagged
    without disturbing the others, huge lambda gives the row mean, a constant row is itself."""
    y = workloads.random_rows(9980 + n, 4, n, "normal", np.float32)
    x, mask, it = run_gpu(tp, y, 0.0, torch.float32)
    assert np.array_equal(x, y) and np.all(it == 0)
    y2 = y.copy()
    y2[1, n // 3] = np.nan
    x, mask, it = run_gpu(tp, y2, 0.5, torch.float32)
    assert it[1] == -2 and np.all(np.isnan(x[1]))
    check_forward(y2[[0, 2, 3]], 0.5, x[[0, 2, 3]], mask[[0, 2, 3]], it[[0, 2, 3]], "f32")
    y64 = y.astype(np.float64)
    lmax = np.abs(np.cumsum(y64 - y64.mean(1, keepdims=True), axis=1)[:, :-1]).max(1)
    x, mask, it = run_gpu(tp, y64, lmax * 1.01, torch.float64)
    np.testing.assert_allclose(x, np.repeat(y64.mean(1, keepdims=True), n, 1), atol=1e-9)
    yc = np.repeat(y[:, :1], n, axis=1)
    x, mask, it = run_gpu(tp, yc, 0.7, torch.float32)
    assert np.abs(x - yc).max() <= 1e-6 * (np.abs(yc).max() + 1)


def test_strided_rows(tp):
    base = workloads.random_rows(9600, 12, 333, "step", np.float32)
    yt = torch.as_tensor(base, device="cuda")[:, :300]      # stride 333 > n = 300
    x, mask, it = tp.tv1d_fwd(yt, 0.4, want_iters=True)
    torch.cuda.synchronize()
    check_forward(base[:, :300], 0.4, x.cpu().numpy(), mask.cpu().numpy(), it.cpu().numpy(), "f32")


def test_empty_batch(tp):
    y = torch.empty((0, 64), device="cuda")
    x, mask, it = tp.tv1d_fwd(y, 0.3, want_iters=True)
    assert x.shape == (0, 64)


def test_autograd(tp):
    rng = np.random.default_rng(9700)
    y = torch.tensor(rng.standard_normal((5, 40)), dtype=torch.float64, device="cuda", requires_grad=True)
    lam = torch.tensor(rng.uniform(0.2, 0.6, 5), dtype=torch.float64, device="cuda", requires_grad=True)
    x = tp.tv1d(y, lam)
    g = torch.tensor(rng.standard_normal((5, 40)), dtype=torch.float64, device="cuda")
    (x * g).sum().backward()
    xr, brk, sgn = oracle.prox1d_batch(y.detach().cpu().numpy(), lam.detach().cpu().numpy())
    gy, gl = oracle.bwd1d_batch(brk, sgn, g.cpu().numpy())
    np.testing.assert_allclose(y.grad.cpu().numpy(), gy, atol=1e-9)
    np.testing.assert_allclose(lam.grad.cpu().numpy(), gl, atol=1e-9)


def test_c2_sampled_full_size(tp):
    """BASELINE configs[1] at full size (65536 x 1024, per-row lam, fp32) in the bench's
    launch configuration; the oracle checks a seeded sample of rows one by one."""
    w = workloads.c2()
    x, mask, it = run_gpu(tp, w.y, w.lam.astype(np.float32), torch.float32)
    assert np.all(it >= 0)
    rows = np.random.default_rng(5).choice(w.y.shape[0], 768, replace=False)
    check_forward(w.y[rows], w.lam[rows], x[rows], mask[rows], it[rows], "f32")
    gt = torch.as_tensor(w.grad, device="cuda")
    gy, gl = tp.tv1d_bwd(gt, torch.as_tensor(mask, device="cuda"), 1)
    torch.cuda.synchronize()
    gy = gy.cpu().numpy()[rows]
    gl = gl.cpu().numpy()[rows]
    brk, sgn = codes_to_brk_sgn(unpack_codes(mask[rows], 1024))
    gy_ref, gl_ref = oracle.bwd1d_batch(brk, sgn, w.grad[rows].astype(np.float64), nthreads=8)
    assert np.abs(gy - gy_ref).max() <= TOL["f32"] * rng_range(w.grad)
    assert np.abs(gl - gl_ref).max() <= TOL["f32"] * (np.abs(gl_ref).max() + 1)
