"""Vectorised fp64 model of the kernel's fast-mode PN (projected full Newton steps from
the partition candidate) to count iterations under different initial bound sets.
Research aid only (not product, not a test)."""
import sys

import numpy as np

sys.path.insert(0, '.')
import oracle  # noqa: E402
from paper_2204_03643_b200 import workloads  # noqa: E402


def candidate(y, u, bnd):
    """Partition candidate of a bound set (bnd[n-1] must be True): xhat, uhat."""
    n = len(y)
    ends = np.flatnonzero(bnd)
    starts = np.concatenate([[0], ends[:-1] + 1])
    ssum = np.add.reduceat(y, starts)
    uR = u[ends]
    uL = np.concatenate([[0.0], uR[:-1]])
    ln = ends - starts + 1
    val = (ssum + uR - uL) / ln
    xh = np.repeat(val, ln)
    # uhat_i = uL + sum_{a..i}(xh - y)
    seg = np.repeat(np.arange(len(ln)), ln)
    c = np.cumsum(xh - y)
    cstart = np.concatenate([[0.0], c[ends[:-1]]])
    uh = uL[seg] + c - cstart[seg]
    return xh, uh


def pn(y, lam, init_pos=None, init_neg=None, maxit=64):
    n = len(y)
    y = y - y.mean()
    pin = np.zeros(n, bool)
    pin[n - 1] = True
    u = np.zeros(n)
    bnd = pin.copy()
    if init_pos is not None:
        u[init_pos] = lam
        u[init_neg] = -lam
        bnd |= init_pos | init_neg
    first = True
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]])
            g = np.append(np.diff(x), 0)
            bnd = pin | ((np.abs(u) >= lam) & (u * g > 0))
        xh, uh = candidate(y, u, bnd)
        free = ~bnd
        feas = np.all(np.abs(uh[free]) <= lam * (1 + 1e-12) + 1e-12)
        jb = bnd & ~pin
        dx = np.append(np.diff(xh), 0)
        sgn = np.all(u[jb] * dx[jb] >= -1e-12)
        if feas and sgn:
            return xh, it + 1
        u = np.where(bnd, u, np.clip(uh, -lam, lam))
        first = False
    return xh, maxit


def coarse_init(y, lam, m):
    """Bound set from the exact prox of the m-block means with lam/m (block-constant restriction)."""
    n = len(y)
    nb = n // m
    yb = y[:nb * m].reshape(nb, m).mean(1)
    xb = oracle.prox1d(yb, lam / m)
    d = np.diff(xb)
    pos = np.zeros(n, bool)
    neg = np.zeros(n, bool)
    e = np.arange(nb - 1) * m + m - 1
    pos[e[d > 0]] = True
    neg[e[d < 0]] = True
    return pos, neg


if __name__ == "__main__":
    w = workloads.c2(batch=256)
    res = {}
    for name in ("cold", "coarse16", "coarse8", "coarse32"):
        its = []
        errs = []
        for b in range(256):
            y = w.y[b].astype(np.float64)
            lam = float(w.lam[b])
            if name == "cold":
                xh, it = pn(y, lam)
            else:
                m = int(name[6:])
                p, q = coarse_init(y, lam, m)
                xh, it = pn(y, lam, p, q)
            ref = oracle.prox1d(y, lam)
            errs.append(np.abs(xh + y.mean() - ref).max())
            its.append(it)
        its = np.array(its)
        print("%-9s iters mean %.2f (even %.2f odd %.2f) p99 %d max %d  maxerr %.1e" % (
            name, its.mean(), its[::2].mean(), its[1::2].mean(), np.percentile(its, 99), its.max(), max(errs)))


def coarse_pn_init(y, lam, m, inner=None):
    """Coarse bound set from PN on the m-block means (lam/m); returns (pos, neg, coarse iters)."""
    n = len(y)
    nb = n // m
    yb = y[:nb * m].reshape(nb, m).mean(1)
    if inner:
        p2, q2, it2 = coarse_pn_init(yb, lam / m, inner)
        xb, itc = pn(yb, lam / m, p2, q2)
    else:
        xb, itc = pn(yb, lam / m)
        it2 = 0
    d = np.diff(xb)
    pos = np.zeros(n, bool)
    neg = np.zeros(n, bool)
    e = np.arange(nb - 1) * m + m - 1
    pos[e[d > 1e-12]] = True
    neg[e[d < -1e-12]] = True
    return pos, neg, (itc, it2)


def run2():
    w = workloads.c2(batch=256)
    for m, inner in ((16, None), (8, None), (4, None), (8, 4), (16, 4), (32, None)):
        its, cits, c2its = [], [], []
        for b in range(256):
            y = w.y[b].astype(np.float64)
            lam = float(w.lam[b])
            p, q, (itc, it2) = coarse_pn_init(y, lam, m, inner)
            xh, it = pn(y, lam, p, q)
            its.append(it); cits.append(itc); c2its.append(it2)
        its = np.array(its)
        print("m=%d inner=%s fine mean %.2f p99 %d max %d | coarse mean %.2f max %d | inner mean %.2f" % (
            m, inner, its.mean(), np.percentile(its, 99), its.max(), np.mean(cits), max(cits), np.mean(c2its)))


def run3():
    """How many fine iterations from perturbed exact bound sets (what a better init could buy)."""
    w = workloads.c2(batch=128)
    for shift in (0, 1, 2, 4, 8):
        its = []
        for b in range(128):
            y = w.y[b].astype(np.float64)
            lam = float(w.lam[b])
            x = oracle.prox1d(y, lam)
            d = np.diff(x)
            n = len(y)
            pos = np.zeros(n, bool); neg = np.zeros(n, bool)
            rng = np.random.default_rng(b)
            for e in np.flatnonzero(np.abs(d) > 0):
                e2 = int(np.clip(e + rng.integers(-shift, shift + 1), 0, n - 2))
                if d[e] > 0: pos[e2] = True
                else: neg[e2] = True
            _, it = pn(y, lam, pos, neg)
            its.append(it)
        its = np.array(its)
        print("exact jumps shifted by <= %d: fine iters mean %.2f max %d" % (shift, its.mean(), its.max()))


def pdas(y, lam, init_pos=None, init_neg=None, maxit=64):
    """Primal-dual active set (semismooth Newton) on the same dual: the next bound set is
    read off the partition candidate itself -- free edges with |uhat| > lam join with the
    sign of uhat, bound edges stay iff the candidate jumps in their direction."""
    n = len(y)
    y = y - y.mean()
    pin = np.zeros(n, bool)
    pin[n - 1] = True
    sp = np.zeros(n, bool) if init_pos is None else init_pos.copy()
    sn = np.zeros(n, bool) if init_neg is None else init_neg.copy()
    for it in range(maxit):
        u = np.where(sp, lam, np.where(sn, -lam, 0.0))
        bnd = pin | sp | sn
        xh, uh = candidate(y, u, bnd)
        dx = np.append(np.diff(xh), 0)
        free = ~bnd
        np_ = (free & (uh > lam * (1 + 1e-12) + 1e-12)) | (sp & (dx > 0))
        nn_ = (free & (uh < -lam * (1 + 1e-12) - 1e-12)) | (sn & (dx < 0))
        np_ &= ~pin
        nn_ &= ~pin
        if np.array_equal(np_, sp) and np.array_equal(nn_, sn):
            return xh, it + 1
        sp, sn = np_, nn_
    return xh, maxit


def run4():
    w = workloads.c2(batch=256)
    for name in ("cold", "coarse16"):
        for solver in ("pn", "pdas"):
            its, errs = [], []
            for b in range(256):
                y = w.y[b].astype(np.float64)
                lam = float(w.lam[b])
                p = q = None
                if name != "cold":
                    p, q, _ = coarse_pn_init(y, lam, 16)
                xh, it = (pn if solver == "pn" else pdas)(y, lam, p, q)
                ref = oracle.prox1d(y, lam)
                errs.append(np.abs(xh + y.mean() - ref).max())
                its.append(it)
            its = np.array(its)
            print("%-9s %-5s iters mean %.2f p99 %d max %d  maxerr %.1e" % (
                name, solver, its.mean(), np.percentile(its, 99), its.max(), max(errs)))
    # shifted exact jumps
    w = workloads.c2(batch=128)
    for shift in (1, 4):
        for solver in ("pn", "pdas"):
            its = []
            for b in range(128):
                y = w.y[b].astype(np.float64)
                lam = float(w.lam[b])
                x = oracle.prox1d(y, lam)
                d = np.diff(x)
                n = len(y)
                pos = np.zeros(n, bool); neg = np.zeros(n, bool)
                rng = np.random.default_rng(b)
                for e in np.flatnonzero(np.abs(d) > 0):
                    e2 = int(np.clip(e + rng.integers(-shift, shift + 1), 0, n - 2))
                    if d[e] > 0: pos[e2] = True
                    else: neg[e2] = True
                _, it = (pn if solver == "pn" else pdas)(y, lam, pos, neg)
                its.append(it)
            its = np.array(its)
            print("shift<=%d %-5s iters mean %.2f max %d" % (shift, solver, its.mean(), its.max()))


def pn_eps(y, lam, init_pos=None, init_neg=None, maxit=64, eps=0.0):
    """PN with Bertsekas' epsilon-active bound set: edges within eps*lam of the bound with an
    outward gradient are bound (snapped to the bound)."""
    n = len(y)
    y = y - y.mean()
    pin = np.zeros(n, bool)
    pin[n - 1] = True
    u = np.zeros(n)
    bnd = pin.copy()
    if init_pos is not None:
        u[init_pos] = lam
        u[init_neg] = -lam
        bnd |= init_pos | init_neg
    first = True
    for it in range(maxit):
        if not first:
            x = y + u - np.concatenate([[0], u[:-1]])
            g = np.append(np.diff(x), 0)
            near = np.abs(u) >= lam * (1 - eps)
            bnd = pin | (near & (u * g > 0))
            u = np.where(bnd & ~pin, np.sign(u) * lam, u)
        xh, uh = candidate(y, u, bnd)
        free = ~bnd
        feas = np.all(np.abs(uh[free]) <= lam * (1 + 1e-12) + 1e-12)
        jb = bnd & ~pin
        dx = np.append(np.diff(xh), 0)
        sgn = np.all(u[jb] * dx[jb] >= -1e-12)
        if feas and sgn:
            return xh, it + 1
        u = np.where(bnd, u, np.clip(uh, -lam, lam))
        first = False
    return xh, maxit


def run5():
    w = workloads.c2(batch=256)
    for eps in (0.0, 0.01, 0.05, 0.1, 0.2, 0.4):
        its, errs = [], []
        for b in range(256):
            y = w.y[b].astype(np.float64)
            lam = float(w.lam[b])
            p, q, _ = coarse_pn_init(y, lam, 16)
            xh, it = pn_eps(y, lam, p, q, eps=eps)
            ref = oracle.prox1d(y, lam)
            errs.append(np.abs(xh + y.mean() - ref).max())
            its.append(it)
        its = np.array(its)
        print("eps %.2f iters mean %.2f p99 %d max %d  maxerr %.1e" % (eps, its.mean(), np.percentile(its, 99),
                                                                     its.max(), max(errs)))


def dykstra_model(X, lam, K=4, prune=False):
    """fp64 model of the staged 2D Dykstra passes with warm starts from the previous
    same-orientation jump set; prune=True drops warm edges whose jump sign disagrees with
    the primal at the previous pass's dual (x(u_{k-1}) = the pass input minus P / Q, i.e.
    the current Y for rows and Z for columns).  Returns per-pass mean PN iterations."""
    H, W = X.shape
    Y = X.copy()
    P = np.zeros_like(X)
    Q = np.zeros_like(X)
    mr = mc = None
    its = []
    for k in range(K):
        A = Y + P
        Z = np.empty_like(X)
        nm = (np.zeros((H, W), bool), np.zeros((H, W), bool))
        itr = []
        for i in range(H):
            p = q = None
            if mr is not None:
                p, q = mr[0][i].copy(), mr[1][i].copy()
                if prune:
                    d = np.append(np.diff(Y[i]), 0)
                    p &= d > 0
                    q &= d < 0
            xh, it = pn(A[i], lam, p, q)
            Z[i] = xh + A[i].mean()
            d = np.append(np.diff(Z[i]), 0)
            nm[0][i] = d > 0
            nm[1][i] = d < 0
            itr.append(it)
        mr = nm
        P = A - Z
        B = Z + Q
        Yn = np.empty_like(X)
        nm = (np.zeros((W, H), bool), np.zeros((W, H), bool))
        itc = []
        for j in range(W):
            p = q = None
            if mc is not None:
                p, q = mc[0][j].copy(), mc[1][j].copy()
                if prune:
                    d = np.append(np.diff(Z[:, j]), 0)
                    p &= d > 0
                    q &= d < 0
            xh, it = pn(B[:, j], lam, p, q)
            Yn[:, j] = xh + B[:, j].mean()
            d = np.append(np.diff(Yn[:, j]), 0)
            nm[0][j] = d > 0
            nm[1][j] = d < 0
            itc.append(it)
        mc = nm
        Q = B - Yn
        Y = Yn
        its += [np.mean(itr), np.mean(itc)]
    return Y, its


def run6(planes=3, H=224):
    w = workloads.c5(N=1, C=3, H=H, W=H, with_grad=False)
    for c in range(min(planes, 3)):
        X = w.X[0, c].astype(np.float64)
        lam = float(w.lam[c])
        Ya, ia = dykstra_model(X, lam)
        Yb, ib = dykstra_model(X, lam, prune=True)
        print("plane %d lam %.3f  warm: %s" % (c, lam, " ".join("%.2f" % v for v in ia)))
        print("             pruned: %s   |dY| %.1e" % (" ".join("%.2f" % v for v in ib), np.abs(Ya - Yb).max()))
