import numpy as np, sys
sys.path.insert(0,'.'); sys.path.insert(0,'scratch')
import oracle, pn_model
from paper_2204_03643_b200 import workloads
def stats(y, lam, dt=np.float32, maxit=64):
    y = y.astype(dt); n = len(y); y = y - y.mean()
    lam_e = np.full(n, lam, dt); lam_e[n-1:] = 0; pin = np.arange(n) >= n-1
    u = np.zeros(n, dt); bnd = pin.copy(); first = True
    out = dict(it=0, clip=0, a1fail=0)
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]]); g = np.append(np.diff(x), 0)
            bnd = pin | ((np.abs(u) >= lam_e) & (u * g > 0))
        xh = pn_model.candidate(y, u, bnd)
        r = 0.0; ok = True; clip = False; uh = np.empty(n, dt)
        for i in range(n):
            t = xh[i]-y[i]; r += t
            if bnd[i]:
                if not pin[i] and u[i]*(xh[i+1]-xh[i]) < 0: ok = False
                uh[i] = u[i]; r = u[i]
            else:
                if abs(r) > lam_e[i]*(1+1e-6): ok = False; clip = True
                uh[i] = r
        out['it'] += 1
        if ok: return out
        if first or not clip:
            u = np.where(bnd, u, np.clip(uh, -lam_e, lam_e))
        else:
            out['clip'] += 1
            d = np.where(bnd, 0, uh - u); x = y + u - np.concatenate([[0], u[:-1]]); g = np.append(np.diff(x), 0)
            alpha = 1.0
            for trial in range(30):
                un = np.clip(u + alpha*d, -lam_e, lam_e); du = un - u; dl = du - np.concatenate([[0], du[:-1]])
                if -0.5*np.sum(dl*(2*x+dl)) >= 1e-4*np.sum(g*du): break
                alpha *= 0.5
            if trial > 0: out['a1fail'] += 1
            u = un
        first = False
    return out
for name, rows in (("C2", workloads.c2(batch=48, with_grad=False)),):
    tot = dict(it=0, clip=0, a1fail=0)
    for r in range(48):
        o = stats(rows.y[r], rows.lam[r])
        for k in tot: tot[k] += o[k]
    print(name, tot)
w = workloads.c5(N=1, with_grad=False)
tot = dict(it=0, clip=0, a1fail=0)
for h in range(0, 224, 8):
    o = stats(w.X[0,1,h], w.lam[1]); 
    for k in tot: tot[k] += o[k]
    o = stats(w.X[0,1,:,h], w.lam[1]);
    for k in tot: tot[k] += o[k]
print("C5 k=1 rows/cols", tot)
