"""GPU parity of the projected line search (row a-7, P:176 / P:188) and the parallel
step search (row f3) as shipped runtime options (tvp_options_t, include/tvprox.h).

The default solver only globalises a projected Newton step with the search from PN
iteration 12 on (DESIGN.md a-7); here ls_after = 2 makes the search guard every step
whose full Newton point leaves the box from the second iteration on, i.e. the method as
the paper writes it.  Each test proves the branch ran: the per-call diagnostics count the
lines that executed at least one line-search pass and the passes themselves, and for 1D
rows the row_iters words carry each line's own pass count (bits 20..27).  Results must
match the oracle exactly as the default path does (the prox does not depend on the
globalisation, only the iteration count does).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2204_03643_b200 import workloads  # noqa: E402
from tests._util import TOL, codes_to_brk_sgn, rng_range, unpack_codes  # noqa: E402
from tests.test_gpu_parity_2d import run_case  # noqa: E402

FLAVOURS = ["backtrack", "parallel"]


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_03643_b200 import tvprox
    return tvprox


def _diag():
    return torch.zeros(4, dtype=torch.int32, device="cuda")


def _check_1d(tp, y, lam, flavour, per_edge=False, dkey="f32"):
    dtype = torch.float32 if dkey == "f32" else torch.float64
    b, n = y.shape
    diag = _diag()
    hist = torch.zeros((1, 128), dtype=torch.int32, device="cuda")
    opts = tp.make_options(line_search=flavour, ls_after=2, diag=diag, iter_hist=hist)
    yt = torch.as_tensor(y, device="cuda")
    lt = lam if np.ndim(lam) == 0 else torch.as_tensor(np.asarray(lam), dtype=dtype, device="cuda")
    x, mask, it = tp.tv1d_fwd(yt, lt, need_mask=True, want_iters=True, opts=opts)
    torch.cuda.synchronize()
    x = x.cpu().numpy().astype(np.float64)
    itn = it.cpu().numpy()
    d = diag.cpu().numpy()
    assert np.all(itn >= 0), "rows not converged"
    lam64 = np.full(b, float(lam)) if np.ndim(lam) == 0 else np.asarray(lam, np.float64)
    xr, brk, sgn = oracle.prox1d_batch(y.astype(np.float64), lam64, per_edge=per_edge, nthreads=8)
    rng = rng_range(y)
    assert np.abs(x - xr).max() <= TOL[dkey] * rng
    gb, gs = codes_to_brk_sgn(unpack_codes(mask.cpu().numpy(), n))
    dis = (gb != brk) | (gs != sgn)
    if dis.any():
        assert np.abs(np.diff(xr, axis=1))[dis].max() <= 10 * TOL[dkey] * rng
    ls = (itn >> 20) & 0xFF
    # the search ran, and the per-row counts agree with the call's counters
    assert d[0] == b
    assert d[1] > 0 and d[2] > 0, "the line search never ran: %s" % d
    assert int((ls > 0).sum()) == d[1] and int(ls.sum()) == d[2]
    assert hist.sum().item() == b
    return d


@pytest.mark.parametrize("flavour", FLAVOURS)
def test_c2_rows(tp, flavour):
    """C2-shaped rows (unit step + noise, per-row softplus lambda), 1024 samples: two warps
    per line, coarse pre-pass, cross-warp reductions of the search."""
    w = workloads.c2(batch=2048, with_grad=False)
    d = _check_1d(tp, w.y, w.lam.astype(np.float32), flavour)
    print(flavour, "C2 diag", d)


@pytest.mark.parametrize("flavour", FLAVOURS)
@pytest.mark.parametrize("n", [56, 200, 300, 2048, 5000])
def test_rows_geometries(tp, flavour, n):
    """Every register geometry of the row solver: 8-lane (E = 7), half-warp (E = 14),
    one warp (E = 16), 4- and 16-warp long rows."""
    y = workloads.random_rows(31000 + n, 256, n, "normal", np.float32)
    lam = np.random.default_rng(n).uniform(0.3, 2.0, 256).astype(np.float32)
    _check_1d(tp, y, lam, flavour)


@pytest.mark.parametrize("flavour", FLAVOURS)
def test_per_edge_and_fp64(tp, flavour):
    rng = np.random.default_rng(5)
    y = workloads.random_rows(32000, 128, 700, "step", np.float32)
    le = rng.uniform(0.0, 1.5, (128, 699)).astype(np.float32)
    _check_1d(tp, y, le, flavour, per_edge=True)
    y64 = workloads.random_rows(32001, 128, 1000, "normal", np.float64)
    _check_1d(tp, y64, rng.uniform(0.3, 2.0, 128), flavour, dkey="f64")


@pytest.mark.parametrize("flavour", FLAVOURS)
@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_2d_configs(tp, flavour, cfg):
    """C3- (fused 56^2 planes), C4- (512^2, lambda 1) and C5-shaped (224^2, per-channel)
    2D Dykstra with the line search from iteration 2 in every row and column pass: forward,
    mask audit and backward parity as in test_gpu_parity_2d, plus proof the search ran."""
    if cfg == "C3":
        w = workloads.c3(N=2, C=16)
    elif cfg == "C4":
        w = workloads.c4(N=1, C=1)
    else:
        w = workloads.c5(N=2)
    lam = w.lam_scalar if w.lam_mode == "scalar" else w.lam.astype(np.float32)
    diag = _diag()
    opts = tp.make_options(line_search=flavour, ls_after=2, diag=diag)
    run_case(tp, w.X, lam, w.lam_mode, w.iters, opts=opts)
    d = diag.cpu().numpy()
    N, C, H, W = w.X.shape
    assert d[0] == w.iters * N * C * (H + W)
    assert d[1] > 0 and d[2] > 0, "the line search never ran: %s" % d
    print(flavour, cfg, "diag", d)


def test_default_vs_search_same_prox(tp):
    """The globalisation changes iteration counts, not the prox: default, backtracking and
    parallel searches agree with each other to the fp32 tolerance on C2-shaped rows."""
    w = workloads.c2(batch=1024, with_grad=False)
    yt = torch.as_tensor(w.y, device="cuda")
    lt = torch.as_tensor(w.lam.astype(np.float32), device="cuda")
    outs = []
    for opts in (None, tp.make_options(line_search="backtrack", ls_after=1),
                 tp.make_options(line_search="parallel", ls_after=1)):
        x, _, it = tp.tv1d_fwd(yt, lt, need_mask=False, want_iters=True, opts=opts)
        outs.append(x.cpu().numpy().astype(np.float64))
        assert (it >= 0).all()
    rng = rng_range(w.y)
    assert np.abs(outs[0] - outs[1]).max() <= 2 * TOL["f32"] * rng
    assert np.abs(outs[0] - outs[2]).max() <= 2 * TOL["f32"] * rng
