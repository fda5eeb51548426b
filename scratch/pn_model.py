"""Sequential numpy model of the kernel's PN algorithm (debug aid, not product)."""
import numpy as np, sys
sys.path.insert(0,'.')
import oracle

def candidate(y, u, bnd):
    n = len(y); x = np.empty(n); a = 0; ul = 0.0
    for i in range(n):
        if bnd[i]:
            x[a:i+1] = (y[a:i+1].sum() - ul + u[i]) / (i + 1 - a)
            ul = u[i]; a = i + 1
    return x

def solve(y, lam, dt=np.float64, slack=True, verbose=False, maxit=64):
    y = y.astype(dt); n = len(y)
    mean = y.mean(); y = y - mean
    lam_e = np.full(n, lam, dt); lam_e[n-1:] = 0
    pin = np.arange(n) >= n - 1
    u = np.zeros(n, dt); bnd = pin.copy(); first = True
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]])
            g = np.append(np.diff(x), 0)
            out = (np.abs(u) >= lam_e) & (u * g > 0)
            bnd = pin | out
        xh = candidate(y, u, bnd)
        # test
        r = 0.0; A = 0.0; ok = True; clip = False; uh = np.empty(n)
        for i in range(n):
            t = xh[i] - y[i]; r += t; A += abs(t)
            if bnd[i]:
                if not pin[i] and u[i] * (xh[i+1] - xh[i]) < 0: ok = False; 
                uh[i] = u[i]; r = u[i]; A = abs(u[i])
            else:
                sl = np.finfo(dt).eps/2 * 34 * A if slack else 0
                if abs(r) > lam_e[i] * (1 + np.finfo(dt).eps) + sl: ok = False
                if abs(r) > lam_e[i]: clip = True
                uh[i] = r
        if verbose: print(it, "ok", ok, "clip", clip, "nbound", bnd.sum(), "err", np.abs(xh + mean - oracle.prox1d(y.astype(np.float64)+mean, lam)).max())
        if ok: return xh + mean, it + 1
        if first or not clip:
            u = np.where(bnd, u, np.clip(uh, -lam_e, lam_e))
        else:
            d = np.where(bnd, 0, uh - u)
            alpha = 1.0
            x = y + u - np.concatenate([[0], u[:-1]])
            g = np.append(np.diff(x), 0)
            for trial in range(30):
                un = np.clip(u + alpha * d, -lam_e, lam_e)
                du = un - u
                dl = du - np.concatenate([[0], du[:-1]])
                gain = -0.5 * np.sum(dl * (2 * x + dl))
                if gain >= 1e-4 * np.sum(g * du): break
                alpha *= 0.5
            if not gain > 0:
                if verbose: print("stall-accept")
                return xh + mean, -(it + 1)
            u = un
        first = False
    return None, maxit

if __name__ == "__main__":
    col = np.load(sys.argv[1])
    ref = oracle.prox1d(col.astype(np.float64), 1.0)
    for dt in (np.float64, np.float32):
        x, it = solve(col, 1.0, dt, verbose=True)
        print(dt.__name__, "iters", it, "err", np.abs(x - ref).max())
