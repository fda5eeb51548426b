import numpy as np, sys
sys.path.insert(0,'.'); sys.path.insert(0,'scratch')
import oracle, pn_model
from paper_2204_03643_b200 import workloads

def solve_warm(y, lam, warm_signs, dt=np.float32, maxit=64):
    # copy of pn_model.solve with a warm start
    y = y.astype(dt); n = len(y); mean = y.mean(); y = y - mean
    lam_e = np.full(n, lam, dt); lam_e[n-1:] = 0
    pin = np.arange(n) >= n - 1
    u = np.where(warm_signs > 0, lam_e, np.where(warm_signs < 0, -lam_e, 0)).astype(dt)
    bnd = pin | (warm_signs != 0)
    first = True
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]])
            g = np.append(np.diff(x), 0)
            bnd = pin | ((np.abs(u) >= lam_e) & (u * g > 0))
        xh = pn_model.candidate(y, u, bnd)
        r = 0.0; ok = True; clip = False; uh = np.empty(n, dt)
        for i in range(n):
            t = xh[i] - y[i]; r += t
            if bnd[i]:
                if not pin[i] and u[i] * (xh[i+1] - xh[i]) < 0: ok = False
                uh[i] = u[i]; r = u[i]
            else:
                if abs(r) > lam_e[i] * (1 + 1e-6): ok = False; clip = True
                uh[i] = r
        if ok: return xh + mean, it + 1
        if first or not clip:
            u = np.where(bnd, u, np.clip(uh, -lam_e, lam_e))
        else:
            d = np.where(bnd, 0, uh - u); x = y + u - np.concatenate([[0], u[:-1]]); g = np.append(np.diff(x), 0)
            alpha = 1.0
            for trial in range(30):
                un = np.clip(u + alpha * d, -lam_e, lam_e); du = un - u; dl = du - np.concatenate([[0], du[:-1]])
                if -0.5 * np.sum(dl * (2 * x + dl)) >= 1e-4 * np.sum(g * du): break
                alpha *= 0.5
            u = un
        first = False
    return None, maxit

w = workloads.c2(batch=64, with_grad=False)
res = {'cold': [], 'chunk32': [], 'chunk64': []}
for r in range(24):
    y = w.y[r].astype(np.float64); lam = w.lam[r]
    ref = oracle.prox1d(y, lam)
    _, it = solve_warm(y, lam, np.zeros(1024)); res['cold'].append(it)
    for C in (32, 64):
        sg = np.zeros(1024)
        for c0 in range(0, 1024, C):
            xl = oracle.prox1d(y[c0:c0+C], lam)
            d = np.sign(np.diff(xl))
            sg[c0:c0+C-1] = d
        x, it = solve_warm(y, lam, sg)
        assert np.abs(x - ref).max() < 1e-4
        res['chunk%d' % C].append(it)
for k, v in res.items(): print(k, np.mean(v), np.max(v))
