import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle
from paper_2204_03643_b200 import tvprox, workloads
w = workloads.c4(with_grad=False)
N, C, H, W = w.X.shape
Xp = w.X.reshape(N * C, H, W)
# find worst plane with the 2D API
Xt = torch.as_tensor(w.X, device='cuda')
Y, _, _ = tvprox.tv2d_fwd(Xt, 1.0, 4)
Yg = Y.cpu().numpy().reshape(N * C, H, W)
errs = []
for p in range(N * C):
    Yr, _ = oracle.prox2d(Xp[p].astype(np.float64), 1.0, 4)
    errs.append(np.abs(Yg[p] - Yr).max())
errs = np.array(errs); p = int(errs.argmax())
print("worst plane", p, "err", errs[p], "range", np.ptp(Xp), "n planes over tol", (errs > 1e-4*np.ptp(Xp)).sum())
# emulate Dykstra with 1D calls, pass by pass, both sides in the same inputs (GPU fp32 state)
X = Xp[p].astype(np.float32)
Yc = X.copy(); P = np.zeros_like(X); Q = np.zeros_like(X)
for k in range(4):
    A = Yc + P if k else X.copy()
    zt, mask, it = tvprox.tv1d_fwd(torch.as_tensor(A, device='cuda'), 1.0, want_iters=True)
    Z = zt.cpu().numpy(); itn = it.cpu().numpy()
    Zr, _, _ = oracle.prox1d_batch(A.astype(np.float64), np.ones(H), nthreads=8)
    e = np.abs(Z - Zr).max(1)
    r = int(e.argmax())
    print("k", k, "rows: max err %.3e at row %d status %s; stalls %d maxit %d" % (e.max(), r, hex(itn[r]), ((itn >> 16) & 1).sum(), itn.max() & 0xffff))
    if e.max() > 1e-5:
        np.save('gpurun_out/bad_row.npy', A[r])
    P = A - Z
    B = Z + Q if k else Z.copy()
    yt, mask, it = tvprox.tv1d_fwd(torch.as_tensor(np.ascontiguousarray(B.T), device='cuda'), 1.0, want_iters=True)
    Yn = yt.cpu().numpy().T; itn = it.cpu().numpy()
    Yr, _, _ = oracle.prox1d_batch(np.ascontiguousarray(B.T).astype(np.float64), np.ones(W), nthreads=8)
    e = np.abs(Yn - Yr.T).max(0)
    c = int(e.argmax())
    print("k", k, "cols: max err %.3e at col %d status %s; stalls %d maxit %d" % (e.max(), c, hex(itn[c]), ((itn >> 16) & 1).sum(), itn.max() & 0xffff))
    if e.max() > 1e-5:
        np.save('gpurun_out/bad_col_k%d.npy' % k, B[:, c])
    Q = B - Yn
    Yc = Yn
