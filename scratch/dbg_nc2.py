import numpy as np, torch, sys, pickle
sys.path.insert(0, '.')
from paper_2204_03643_b200 import tvprox, workloads
cfg = sys.argv[1]
w = {"c3": lambda: workloads.c3(with_grad=False), "c5": lambda: workloads.c5(with_grad=False), "c4": lambda: workloads.c4(with_grad=False)}[cfg]()
N, C, H, W = w.X.shape
P = N * C
lamp = np.tile(w.lam, N) if w.lam_mode == "channel" else np.full(P, w.lam_scalar)
X = torch.as_tensor(w.X.reshape(P, H, W), device='cuda')
lam_rows = torch.as_tensor(np.repeat(lamp, H).astype(np.float32), device='cuda')
lam_cols = torch.as_tensor(np.repeat(lamp, W).astype(np.float32), device='cuda')
Y = X.clone(); Pd = torch.zeros_like(X); Q = torch.zeros_like(X)
rm = cm = None; saved = []
for k in range(4):
    A = (Y + Pd) if k else X.clone()
    z, mask, it = tvprox.tv1d_fwd(A.reshape(P * H, W), lam_rows, want_iters=True, warm_mask=rm)
    itn = it.cpu().numpy()
    bad = np.where(itn < 0)[0]
    print("k", k, "rows nonconv", len(bad), "stall", ((itn >> 16) & 1).sum(), "max", (itn & 0xffff).max(), "mean %.2f" % (itn & 0xffff).mean(), "hist", np.bincount(itn & 0xffff)[:8].tolist())
    for r in bad[:3]:
        saved.append(dict(kind='row', k=k, y=A.reshape(P*H, W)[r].cpu().numpy(), lam=float(lam_rows[r]), warm=None if rm is None else rm[r].cpu().numpy()))
    rm = mask
    Z = z.reshape(P, H, W)
    Pd = A - Z
    B = (Z + Q) if k else Z.clone()
    Bt = B.transpose(1, 2).contiguous().reshape(P * W, H)
    yt, mask, it = tvprox.tv1d_fwd(Bt, lam_cols, want_iters=True, warm_mask=cm)
    itn = it.cpu().numpy()
    bad = np.where(itn < 0)[0]
    print("k", k, "cols nonconv", len(bad), "stall", ((itn >> 16) & 1).sum(), "max", (itn & 0xffff).max(), "mean %.2f" % (itn & 0xffff).mean(), "hist", np.bincount(itn & 0xffff)[:8].tolist())
    for c in bad[:3]:
        saved.append(dict(kind='col', k=k, y=Bt[c].cpu().numpy(), lam=float(lam_cols[c]), warm=None if cm is None else cm[c].cpu().numpy()))
    cm = mask
    Yn = yt.reshape(P, W, H).transpose(1, 2)
    Q = B - Yn
    Y = Yn.contiguous()
pickle.dump(saved, open('gpurun_out/nc_%s.pkl' % cfg, 'wb'))
