import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle
from paper_2204_03643_b200 import tvprox, workloads
cfg = sys.argv[1]
w = {"c3": lambda: workloads.c3(N=8, with_grad=False), "c5": lambda: workloads.c5(N=8, with_grad=False)}[cfg]()
N, C, H, W = w.X.shape
lamp = np.tile(w.lam, N) if w.lam_mode == "channel" else np.full(N*C, w.lam_scalar)
saved = []
for p in range(N * C):
    X = w.X.reshape(N * C, H, W)[p]
    lam = float(np.float32(lamp[p]))
    Yc = X.copy(); P = np.zeros_like(X); Q = np.zeros_like(X)
    rm = None; cm = None
    for k in range(4):
        A = Yc + P if k else X.copy()
        zt, mask, it = tvprox.tv1d_fwd(torch.as_tensor(A, device='cuda'), lam, want_iters=True, warm_mask=rm)
        Z = zt.cpu().numpy(); itn = it.cpu().numpy()
        for r in np.where(itn < 0)[0][:2]:
            saved.append((A[r].copy(), lam, 'row', p, k, rm[r].cpu().numpy() if rm is not None else None))
        rm = mask
        P = A - Z
        B = Z + Q if k else Z.copy()
        yt, mask, it = tvprox.tv1d_fwd(torch.as_tensor(np.ascontiguousarray(B.T), device='cuda'), lam, want_iters=True, warm_mask=cm)
        Yn = yt.cpu().numpy().T; itn = it.cpu().numpy()
        for c in np.where(itn < 0)[0][:2]:
            saved.append((B[:, c].copy(), lam, 'col', p, k, cm[c].cpu().numpy() if cm is not None else None))
        cm = mask
        Q = B - Yn
        Yc = Yn
    if len(saved) >= 6: break
import pickle
pickle.dump(saved, open('gpurun_out/nc_%s.pkl' % cfg, 'wb'))
print("nonconverged lines found:", len(saved))
np.save('gpurun_out/nc_lines_%s.npy' % cfg, np.array([s[0] for s in saved]))
np.save('gpurun_out/nc_lams_%s.npy' % cfg, np.array([s[1] for s in saved]))
print([s[2:5] for s in saved])
