import numpy as np, sys
sys.path.insert(0,'.'); sys.path.insert(0,'scratch')
import oracle, pn_model
from paper_2204_03643_b200 import workloads
def run(y, lam, use_ls, dt=np.float32, maxit=64):
    y0=y; y = y.astype(dt); n = len(y); mean=y.mean(); y = y - mean
    lam_e = np.full(n, lam, dt); lam_e[n-1:] = 0; pin = np.arange(n) >= n-1
    u = np.zeros(n, dt); bnd = pin.copy(); first = True; hist=[]
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]]); g = np.append(np.diff(x), 0)
            bnd = pin | ((np.abs(u) >= lam_e) & (u * g > 0))
        key=bnd.tobytes()
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
        if ok: return it+1, xh+mean
        if first or not clip or not use_ls:
            u = np.where(bnd, u, np.clip(uh, -lam_e, lam_e))
        else:
            d = np.where(bnd, 0, uh - u); x = y + u - np.concatenate([[0], u[:-1]]); g = np.append(np.diff(x), 0)
            alpha = 1.0
            for trial in range(30):
                un = np.clip(u + alpha*d, -lam_e, lam_e); du = un - u; dl = du - np.concatenate([[0], du[:-1]])
                if -0.5*np.sum(dl*(2*x+dl)) >= 1e-4*np.sum(g*du): break
                alpha *= 0.5
            u = un
        first = False
    return maxit, None
w = workloads.c2(batch=200, with_grad=False)
for use_ls in (True, False):
    its=[]; fails=0; errs=[]
    for r in range(100):
        it, x = run(w.y[r], w.lam[r], use_ls); its.append(it)
        if x is None: fails+=1
        else: errs.append(np.abs(x-oracle.prox1d(w.y[r].astype(np.float64), w.lam[r])).max())
    print("LS" if use_ls else "noLS", "mean it", np.mean(its), "max", np.max(its), "fails", fails, "maxerr", max(errs))
rng=np.random.default_rng(0)
for name, gen in (("iid n=56", lambda: rng.standard_normal(56)), ("iid n=224", lambda: rng.standard_normal(224)),
                  ("relu n=56", lambda: np.maximum(rng.standard_normal(56),0)), ("iid n=512", lambda: rng.standard_normal(512)),
                  ("rect512", lambda: workloads.rect_planes(rng, 1, 1, 512)[0,0])):
    for use_ls in (True, False):
        its=[]; fails=0
        for t in range(150):
            y=gen(); lam=rng.choice([0.05,0.2,0.7,1.5,4.0])
            it,x=run(y,lam,use_ls); its.append(it); fails+= x is None
        print(name, "LS" if use_ls else "noLS", "mean", np.mean(its), "max", max(its), "fails", fails)
