"""GPU determinism and shard independence (DESIGN.md section 2 / SURVEY 8(b), 8(e)).

* Run to run: the same call on the same inputs gives bitwise the same outputs, masks and
  lambda gradients (no float atomics; fixed-order reductions).
* Shard independence: rows (1D) and planes (2D) are independent problems, so a
  batch computed in pieces -- what a rank of the multi-GPU run computes -- is bitwise the
  slice of the whole batch's result.  This holds even where two lines share a warp: a
  line that has stopped reproduces its candidate bitwise while its partner iterates.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2204_03643_b200 import workloads  # noqa: E402


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_03643_b200 import _lib, tvprox
    return tvprox, _lib


def _rows(n, batch, seed):
    y = workloads.random_rows(seed, batch, n, "step", np.float32)
    lam = np.random.default_rng(seed + 1).uniform(0.1, 1.5, batch).astype(np.float32)
    g = np.random.default_rng(seed + 2).standard_normal((batch, n)).astype(np.float32)
    return (torch.as_tensor(y, device="cuda"), torch.as_tensor(lam, device="cuda"),
            torch.as_tensor(g, device="cuda"))


@pytest.mark.parametrize("n", [56, 100, 224, 512, 1024, 3000])
def test_1d_run_to_run_bitwise(tp, n):
    tvprox, lib = tp
    y, lam, g = _rows(n, 257, 9100 + n)
    outs = []
    for _ in range(2):
        x, mask, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
        gy, gl = tvprox.tv1d_bwd(g, mask, lib.LAM_PER_ROW, want_lam=True)
        xs, ms, _ = tvprox.tv1d_fwd(y, 0.7, want_iters=True)
        gys, gls = tvprox.tv1d_bwd(g, ms, lib.LAM_SCALAR, want_lam=True)
        outs.append([t.cpu() for t in (x, mask, it, gy, gl, xs, ms, gys, gls)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n", [56, 100, 224, 512, 1024])
def test_1d_shard_equals_slice(tp, n):
    tvprox, lib = tp
    y, lam, g = _rows(n, 301, 9200 + n)
    x, mask, it = tvprox.tv1d_fwd(y, lam, want_iters=True)
    gy, gl = tvprox.tv1d_bwd(g, mask, lib.LAM_PER_ROW, want_lam=True)
    for a, b in ((0, 77), (77, 78), (78, 301), (1, 300)):
        xa, ma, ita = tvprox.tv1d_fwd(y[a:b].contiguous(), lam[a:b].contiguous(), want_iters=True)
        gya, gla = tvprox.tv1d_bwd(g[a:b].contiguous(), ma, lib.LAM_PER_ROW, want_lam=True)
        assert torch.equal(xa, x[a:b]) and torch.equal(ma, mask[a:b]) and torch.equal(ita, it[a:b])
        assert torch.equal(gya, gy[a:b]) and torch.equal(gla, gl[a:b])


@pytest.mark.parametrize("shape", [(6, 3, 224, 224), (5, 4, 56, 56), (3, 2, 100, 130)])
def test_2d_shard_equals_slice(tp, shape):
    tvprox, lib = tp
    N, C, H, W = shape
    rng = np.random.default_rng(9300 + H)
    X = torch.as_tensor(rng.standard_normal(shape).astype(np.float32), device="cuda")
    G = torch.as_tensor(rng.standard_normal(shape).astype(np.float32), device="cuda")
    lam = torch.as_tensor(np.linspace(0.2, 1.3, C).astype(np.float32), device="cuda")
    Y, saved, _ = tvprox.tv2d_fwd(X, lam, 4, training=True)
    GX, _ = tvprox.tv2d_bwd(G, saved, lib.LAM_PER_CHANNEL, 4, want_lam=True)
    Y2, saved2, _ = tvprox.tv2d_fwd(X, lam, 4, training=True)
    GX2, _ = tvprox.tv2d_bwd(G, saved2, lib.LAM_PER_CHANNEL, 4, want_lam=True)
    assert torch.equal(Y, Y2) and torch.equal(saved, saved2) and torch.equal(GX, GX2)
    for a, b in ((0, 1), (1, N - 1), (N - 1, N)):
        Ya, sa, _ = tvprox.tv2d_fwd(X[a:b].contiguous(), lam, 4, training=True)
        GXa, _ = tvprox.tv2d_bwd(G[a:b].contiguous(), sa, lib.LAM_PER_CHANNEL, 4, want_lam=True)
        assert torch.equal(Ya, Y[a:b])
        assert torch.equal(GXa, GX[a:b])
