"""GPU parity of the TV layer pieces (NEXT f1, Sec. 3.1 / Fig. 2) vs the oracle:
rows-only / columns-only spatial modes, SoftPlus lambda (Eq. 3), sharpening
(Eq. 4), the lambda = 0 identity of both modes, and the layer's gradients."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from tests._util import TOL, codes_to_brk_sgn, rng_range, unpack_codes  # noqa: E402


@pytest.fixture(scope="module")
def mods():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_03643_b200 import layer, tvprox
    return tvprox, layer


def _lines_ref(X, lamp, axis):
    """Oracle: 1D prox per row (axis 0) or column (axis 1) of every plane."""
    P, H, W = X.shape
    Y = np.empty_like(X)
    for p in range(P):
        A = X[p] if axis == 0 else X[p].T
        y, _, _ = oracle.prox1d_batch(A, np.full(A.shape[0], lamp[p]))
        Y[p] = y if axis == 0 else y.T
    return Y


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("H,W", [(5, 37), (56, 56), (33, 600), (224, 40)])
def test_lines_forward_backward(mods, axis, H, W):
    tp, _ = mods
    rng = np.random.default_rng(H * 7 + W + axis)
    X = rng.standard_normal((2, 3, H, W)).astype(np.float32)
    lam = np.array([0.2, 0.5, 1.1], np.float32)
    Xt = torch.as_tensor(X, device="cuda")
    Y, mask = tp.tv2d_lines_fwd(Xt, torch.as_tensor(lam, device="cuda"), axis)
    torch.cuda.synchronize()
    lamp = np.tile(lam.astype(np.float64), 2)
    Yr = _lines_ref(X.reshape(6, H, W).astype(np.float64), lamp, axis)
    assert np.abs(Y.cpu().numpy().reshape(6, H, W) - Yr).max() <= TOL["f32"] * rng_range(X)
    G = rng.standard_normal(X.shape).astype(np.float32)
    GX, gl = tp.tv2d_lines_bwd(torch.as_tensor(G, device="cuda"), mask, 3, axis)
    torch.cuda.synchronize()
    n = W if axis == 0 else H
    brk, sgn = codes_to_brk_sgn(unpack_codes(mask.cpu().numpy(), n))
    Gl = G.reshape(6, H, W).astype(np.float64)
    Gl = Gl if axis == 0 else Gl.transpose(0, 2, 1)
    gy, glr = oracle.bwd1d_batch(brk, sgn, np.ascontiguousarray(Gl.reshape(-1, n)))
    gy = gy.reshape(Gl.shape)
    gy = gy if axis == 0 else gy.transpose(0, 2, 1)
    assert np.abs(GX.cpu().numpy().reshape(6, H, W) - gy).max() <= TOL["f32"] * rng_range(G)
    ref = glr.reshape(2, 3, -1).sum(axis=(0, 2))
    assert np.abs(gl.cpu().numpy() - ref).max() <= TOL["f32"] * (np.abs(glr).sum() + 1)


def test_softplus_and_axpby(mods):
    tp, _ = mods
    t = torch.linspace(-30, 30, 1001, dtype=torch.float64, device="cuda")
    lam = tp.softplus_fwd(t).cpu().numpy()
    tn = t.cpu().numpy()
    np.testing.assert_allclose(lam, np.log1p(np.exp(-np.abs(tn))) + np.maximum(tn, 0), rtol=1e-14, atol=1e-300)
    g = torch.ones_like(t)
    np.testing.assert_allclose(tp.softplus_bwd(t, g).cpu().numpy(), 1 / (1 + np.exp(-tn)), rtol=1e-14)
    x = torch.arange(10, dtype=torch.float32, device="cuda")
    y = torch.ones(10, dtype=torch.float32, device="cuda")
    tp.axpby_(x, y, 2.0, -1.0)
    np.testing.assert_array_equal(y.cpu().numpy(), 2 * np.arange(10) - 1)


@pytest.mark.parametrize("mode", ["2d", "rows", "cols"])
@pytest.mark.parametrize("sharp", [False, True])
def test_layer_forward_and_grads(mods, mode, sharp):
    tp, layer = mods
    rng = np.random.default_rng(3)
    X = rng.standard_normal((2, 3, 12, 10))
    lt = np.array([-1.0, 0.0, 0.7])
    L = layer.TVLayer(3, is_sharp=sharp, mode=mode, iters=3, dtype=torch.float64, device="cuda")
    with torch.no_grad():
        L._lmbd.copy_(torch.as_tensor(lt))
    Xt = torch.as_tensor(X, device="cuda").requires_grad_(True)
    Y = L(Xt)
    G = rng.standard_normal(X.shape)
    (Y * torch.as_tensor(G, device="cuda")).sum().backward()
    lam = np.log1p(np.exp(lt))
    lamp = np.tile(lam, 2)
    Xp = X.reshape(6, 12, 10)
    if mode == "2d":
        Pr, segs = oracle.prox2d_batch(Xp, lamp, 3)
        gP, glp = oracle.bwd2d_batch(segs, G.reshape(6, 12, 10) * (-1.0 if sharp else 1.0), 3)
    else:
        axis = 0 if mode == "rows" else 1
        Pr = _lines_ref(Xp, lamp, axis)
        # VJP through the oracle segmentation of the 1D solutions
        Gs = G.reshape(6, 12, 10) * (-1.0 if sharp else 1.0)
        gP = np.empty_like(Gs)
        glp = np.zeros(6)
        for p in range(6):
            A = Pr[p] if axis == 0 else Pr[p].T
            Gp = Gs[p] if axis == 0 else Gs[p].T
            out = np.empty_like(A)
            for i in range(A.shape[0]):
                b, s = oracle.codes(A[i], lamp[p])
                out[i], _, t = oracle.bwd1d(b, s, Gp[i])
                glp[p] += t
            gP[p] = out if axis == 0 else out.T
    Yr = 2 * Xp - Pr if sharp else Pr
    np.testing.assert_allclose(Y.detach().cpu().numpy().reshape(6, 12, 10), Yr, atol=1e-9)
    gX = 2 * G.reshape(6, 12, 10) + gP if sharp else gP
    np.testing.assert_allclose(Xt.grad.cpu().numpy().reshape(6, 12, 10), gX, atol=1e-9)
    glam = glp.reshape(2, 3).sum(0)
    sig = 1 / (1 + np.exp(-lt))
    np.testing.assert_allclose(L._lmbd.grad.cpu().numpy(), glam * sig, atol=1e-9)


def test_layer_identity_at_zero_lambda(mods):
    """lambda = 0 makes both modes the identity; SoftPlus(t) -> 0 as t -> -inf."""
    tp, layer = mods
    X = torch.randn(2, 3, 9, 11, device="cuda")
    for sharp in (False, True):
        L = layer.TVLayer(3, is_sharp=sharp, init=-200.0, device="cuda")
        Y = L(X)
        assert torch.equal(Y, X) or torch.allclose(Y, X, atol=0, rtol=0)


def test_per_edge_lambda_grad_layouts(mods):
    """A per-edge lambda given as [batch, n] (the last column unused) gets a gradient of the
    same shape with zeros there; a CPU lambda gets its gradient on the CPU."""
    tp, _ = mods
    rng = np.random.default_rng(12)
    y = torch.tensor(rng.standard_normal((6, 40)), device="cuda", requires_grad=True)
    lam_full = torch.tensor(rng.uniform(0.1, 1.0, (6, 40)), device="cuda", requires_grad=True)
    x = tp.tv1d(y, lam_full)
    g = torch.tensor(rng.standard_normal((6, 40)), device="cuda")
    (x * g).sum().backward()
    assert lam_full.grad.shape == (6, 40)
    assert torch.all(lam_full.grad[:, -1] == 0)
    # same values as the [batch, n-1] form
    lam_e = lam_full.detach()[:, :39].clone().requires_grad_(True)
    y2 = y.detach().clone().requires_grad_(True)
    (tp.tv1d(y2, lam_e) * g).sum().backward()
    assert torch.allclose(lam_full.grad[:, :39], lam_e.grad)
    # CPU per-row lambda: gradient comes back on the CPU, same values
    lam_cpu = torch.tensor(rng.uniform(0.1, 1.0, 6), requires_grad=True)
    y3 = y.detach().clone().requires_grad_(True)
    (tp.tv1d(y3, lam_cpu) * g).sum().backward()
    assert lam_cpu.grad.device.type == "cpu" and lam_cpu.grad.shape == (6,)
    lam_gpu = lam_cpu.detach().cuda().requires_grad_(True)
    (tp.tv1d(y.detach(), lam_gpu) * g).sum().backward()
    assert torch.allclose(lam_cpu.grad, lam_gpu.grad.cpu())
    # 2D, CPU per-channel lambda
    X = torch.tensor(rng.standard_normal((2, 3, 20, 30)), device="cuda", requires_grad=True)
    lc = torch.tensor([0.2, 0.4, 0.8], requires_grad=True)
    (tp.tv2d(X, lc, iters=2) * torch.ones_like(X[:1])).sum().backward()
    assert lc.grad.device.type == "cpu" and lc.grad.shape == (3,)


def test_layer_default_init_and_shared_lambda(mods):
    """TVLayer initialises lambda = 0.05; shared=True learns one lambda for all
    channels ("lambda shared across channels") through the per-channel kernels."""
    tp, layer = mods
    L = layer.TVLayer(num_chan=4, device="cuda")
    assert torch.allclose(L.lam, torch.full((4,), 0.05, device="cuda"), atol=1e-6)
    Ls = layer.TVLayer(num_chan=4, shared=True, init=0.3, dtype=torch.float64, device="cuda")
    assert Ls._lmbd.shape == (1,)
    rng = np.random.default_rng(3)
    X = torch.tensor(rng.standard_normal((2, 4, 24, 24)), device="cuda", requires_grad=True)
    Y = Ls(X)
    G = torch.tensor(rng.standard_normal(Y.shape), device="cuda")
    (Y * G).sum().backward()
    lam = float(np.log1p(np.exp(0.3)))
    Yr, segs = oracle.prox2d_batch(X.detach().cpu().numpy().reshape(8, 24, 24), np.full(8, lam), 4)
    assert np.abs(Y.detach().cpu().numpy().reshape(8, 24, 24) - Yr).max() <= 1e-9 * rng_range(Yr)
    _, glr = oracle.bwd2d_batch(segs, G.cpu().numpy().reshape(8, 24, 24), 4)
    sig = 1.0 / (1.0 + np.exp(-0.3))
    assert abs(Ls._lmbd.grad.item() - glr.sum() * sig) <= 1e-9 * (np.abs(glr).sum() + 1)
