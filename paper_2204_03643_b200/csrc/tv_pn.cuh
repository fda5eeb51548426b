// tv_pn.cuh -- warp-cooperative projected-Newton solver for one 1D TV prox line
// (arXiv 2204.03643, Sec. 3.2 "Forward Operation") and the
// segment-mean backward line primitive (Eq. 7-8).
//
// Dual problem (Eq. 5):  max_u phi(u) = -1/2 ||D^T u||^2 + u^T D y,
// |u_i| <= lam_i, primal x(u) = y - D^T u, gradient g = D x(u).
// Projected Newton (Bertsekas 1982): bound set B = pinned edges plus
// edges at a bound whose gradient points outward; the Newton system Eq. 6
// H_F d_F = g_F with H = D D^T (tridiagonal) is solved on the free set F.
//
// B200 realisation of the Eq. 6 solve: restricted
// to F, D D^T splits into one tridiag(-1,2,-1) block per maximal free run, and
// the full Newton step lands on the face maximiser, whose primal is constant on
// each segment between bound edges:
//     xhat = (sum_{j=a}^{b-1} y_j + u_{b-1} - u_{a-1}) / (b - a)   on [a, b)
// with u at the segment's bound edges (0 at the line ends).  Its dual is the
// running sum uhat_i = u_{a-1} + sum_{j=a}^{i} (xhat_j - y_j), so d = uhat - u.
// On a warp this is two segmented scans plus one reverse broadcast, entirely in
// registers (no 3xN band storage, no Cholesky factor).
#pragma once
#include "tv_common.cuh"

namespace tvp {

template <int W> struct Log2 { static constexpr int v = 1 + Log2<W / 2>::v; };
template <> struct Log2<1> { static constexpr int v = 0; };

// Per-lane view of lambda: one value per line, or one per edge held in registers.
template <typename T, int E, bool PE>
struct Lam {
    T r;
    T e[PE ? E : 1];
    __device__ __forceinline__ T at(int k) const { return PE ? e[PE ? k : 0] : r; }
};

// ---------------------------------------------------------------------------
// Eq. 6 partition solve: w <- xhat for bound set `bnd` (segments end at bound
// edges; u holds the bound values +-lam on them, 0 on pinned edges).
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR>
__device__ __forceinline__ void pn_candidate(const T (&y)[E], const T (&u)[E], uint32_t bnd,
                                             T (&w)[E], int l) {
    // pass 1: lane aggregate of the segment left open at the lane's end
    T s = T(0), ub = T(0);
    int c = 0;
    bool f = false;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        s += y[k];
        c += 1;
        if ((bnd >> k) & 1u) { f = true; ub = u[k]; s = T(0); c = 0; }
    }
    // segmented inclusive scan over the group: (sum, count, left bound value)
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
        T s2 = shup<LPR>(s, d);
        T ub2 = shup<LPR>(ub, d);
        int cf2 = shup<LPR>(c | (f ? (1 << 30) : 0), d);
        if (l >= d && !f) { s += s2; ub = ub2; c += cf2 & 0x3fffffff; f = (cf2 >> 30) & 1; }
    }
    T cs = shup<LPR>(s, 1), cub = shup<LPR>(ub, 1);
    int cc = shup<LPR>(c, 1);
    if (l == 0) { cs = T(0); cub = T(0); cc = 0; }
    // pass 2: segment values at segment ends
    s = cs; c = cc; ub = cub;
    T first = T(0);
    bool hf = false;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        s += y[k];
        c += 1;
        if ((bnd >> k) & 1u) {
            T v = div_count(s + u[k] - ub, c);
            w[k] = v;
            if (!hf) first = v;
            hf = true;
            ub = u[k]; s = T(0); c = 0;
        }
    }
    // pass 3: reverse broadcast of each segment's value to its elements
    T v = first;
    bool fv = hf;
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
        T v2 = shdn<LPR>(v, d);
        int f2 = shdn<LPR>((int)fv, d);
        if (l + d < LPR && !fv) { v = v2; fv = f2 != 0; }
    }
    T cur = shdn<LPR>(v, 1);
#pragma unroll
    for (int k = E - 1; k >= 0; --k) {
        if ((bnd >> k) & 1u) cur = w[k]; else w[k] = cur;
    }
}

// ---------------------------------------------------------------------------
// Duality-gap / KKT stop test of the candidate (w = xhat on entry) and Newton
// direction (w = d on exit).  At the candidate the duality gap is
// sum_{i in B} (lam_i |dx_i| - u_i dx_i), zero iff every bound edge's jump has
// the sign of u_i, and the candidate is dual feasible iff |uhat_i| <= lam_i on
// free edges (tested with a summation-error slack; bound edges are never
// feasibility-tested, their uhat only echoes rounding -- DESIGN.md O8).
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR, bool PE>
__device__ __forceinline__ bool pn_test_direction(const T (&y)[E], const T (&u)[E], uint32_t bnd,
                                                  uint32_t pin, T (&w)[E], const Lam<T, E, PE>& lam,
                                                  int l) {
    T r = T(0), A = T(0);
    bool f = false;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        T t = w[k] - y[k];
        r += t;
        A += fabs(t);
        if ((bnd >> k) & 1u) { r = u[k]; A = fabs(u[k]); f = true; }
    }
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
        T r2 = shup<LPR>(r, d), A2 = shup<LPR>(A, d);
        int f2 = shup<LPR>((int)f, d);
        if (l >= d && !f) { r += r2; A += A2; f = f2 != 0; }
    }
    T cr = shup<LPR>(r, 1), cA = shup<LPR>(A, 1);
    if (l == 0) { cr = T(0); cA = T(0); }
    T xnext = shdn<LPR>(w[0], 1);
    constexpr T C = T(E + 2 * Log2<LPR>::v + 8);
    const T eps = Num<T>::eps;
    bool ok = true;
    r = cr; A = cA;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        T xk = w[k];
        T xk1 = (k + 1 < E) ? w[(k + 1 < E) ? k + 1 : k] : xnext;
        T t = xk - y[k];
        r += t;
        A += fabs(t);
        if ((bnd >> k) & 1u) {
            if (!((pin >> k) & 1u)) ok = ok && (u[k] * (xk1 - xk) >= T(0));
            w[k] = T(0);
            r = u[k];
            A = fabs(u[k]);
        } else {
            T lk = lam.at(k);
            ok = ok && (fabs(r) <= lk + eps * (T(2) * lk + C * A));
            w[k] = r - u[k];
        }
    }
    return group_all<LPR>(ok);
}

// Bound set at u: pinned edges plus edges at +-lam whose gradient g = D x(u)
// points out of the box (exact comparison: u is clipped exactly to +-lam).
template <typename T, int E, int LPR, bool PE>
__device__ __forceinline__ uint32_t pn_bound_set(const T (&y)[E], const T (&u)[E], uint32_t pin,
                                                 const Lam<T, E, PE>& lam, int l) {
    T uprev = shup<LPR>(u[E - 1], 1);
    if (l == 0) uprev = T(0);
    T y0n = shdn<LPR>(y[0], 1), u0n = shdn<LPR>(u[0], 1);
    T xk = y[0] + u[0] - uprev;
    uint32_t b = pin;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        T xk1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                            : (y0n + u0n - u[k]);
        T g = xk1 - xk;
        T lk = lam.at(k);
        bool out = (u[k] >= lk && g > T(0)) || (u[k] <= -lk && g < T(0));
        b |= (out ? 1u : 0u) << k;
        xk = xk1;
    }
    return b;
}

// Projected line search along u(alpha) = clip(u + alpha d):
// Armijo  phi(u(alpha)) - phi(u) >= sigma g^T (u(alpha) - u), sigma = 1e-4,
// with quadratic-interpolation backtracking safeguarded to [0.1, 0.5] alpha.
// phi(u(alpha)) - phi(u) = -1/2 sum_j delta_j (2 x_j + delta_j), delta = x(u(alpha)) - x(u),
// evaluated in this difference form for accuracy.  Applies the accepted step to u
// on `run` groups.  Returns true iff the step changed u (group-uniform).
template <typename T, int E, int LPR, bool PE>
__device__ __forceinline__ bool pn_line_search(const T (&y)[E], T (&u)[E], const T (&d)[E],
                                               uint32_t bnd, const Lam<T, E, PE>& lam, int l,
                                               bool run) {
    T uprev = shup<LPR>(u[E - 1], 1);
    if (l == 0) uprev = T(0);
    T y0n = shdn<LPR>(y[0], 1), u0n = shdn<LPR>(u[0], 1);
    T slope = T(0);
    {
        T xk = y[0] + u[0] - uprev;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            T xk1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                                : (y0n + u0n - u[k]);
            slope = fma(xk1 - xk, d[k], slope);
            xk = xk1;
        }
    }
    slope = group_sum<LPR>(slope);
    T alpha = T(1);
    bool pending = run, accepted = false, changed = false;
    for (int trial = 0; trial < 40; ++trial) {
        if (!__any_sync(FULL, pending)) break;
        T lk = lam.at(E - 1);
        T dlast = ((bnd >> (E - 1)) & 1u) ? T(0) : clampv(u[E - 1] + alpha * d[E - 1], -lk, lk) - u[E - 1];
        T duprev = shup<LPR>(dlast, 1);
        if (l == 0) duprev = T(0);
        T F = T(0), G = T(0);
        bool ch = false;
        T xk = y[0] + u[0] - uprev;
#pragma unroll
        for (int k = 0; k < E; ++k) {
            T lk2 = lam.at(k);
            T du = ((bnd >> k) & 1u) ? T(0) : clampv(u[k] + alpha * d[k], -lk2, lk2) - u[k];
            T xk1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                                : (y0n + u0n - u[k]);
            T dl = du - duprev;
            F = fma(dl, T(2) * xk + dl, F);
            G = fma(xk1 - xk, du, G);
            ch = ch || (du != T(0));
            duprev = du;
            xk = xk1;
        }
        F = group_sum<LPR>(F);
        G = group_sum<LPR>(G);
        ch = group_any<LPR>(ch);
        if (pending) {
            T gain = T(-0.5) * F;
            if (gain >= T(1e-4) * G) {
                pending = false; accepted = true; changed = ch;
            } else {
                T den = T(2) * (slope * alpha - gain);
                T an = den > T(0) ? slope * alpha * alpha / den : T(0.5) * alpha;
                alpha = clampv(an, T(0.1) * alpha, T(0.5) * alpha);
                if (alpha < T(1e-12)) pending = false;
            }
        }
    }
    if (accepted && changed) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
            T lk = lam.at(k);
            if (!((bnd >> k) & 1u)) u[k] = clampv(u[k] + alpha * d[k], -lk, lk);
        }
    }
    return accepted && changed;
}

// Full solve of one line per group.  y: centred samples; u: dual (in/out);
// w: output x (centred).  pin: pinned edges.  warm_pos/warm_neg: edges that
// were up/down jumps in a previous solve (warm start, DESIGN.md a-11).
// Returns the per-line status (iterations | stall flag, or -1).
template <typename T, int E, int LPR, bool PE>
__device__ __forceinline__ int pn_solve(const T (&y)[E], T (&u)[E], T (&w)[E], uint32_t pin,
                                        uint32_t warm_pos, uint32_t warm_neg,
                                        const Lam<T, E, PE>& lam, int l, bool active) {
    warm_pos &= ~pin;
    warm_neg &= ~pin;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        T lk = lam.at(k);
        u[k] = ((warm_pos >> k) & 1u) ? lk : (((warm_neg >> k) & 1u) ? -lk : T(0));
    }
    uint32_t bnd = pin | warm_pos | warm_neg;
    // iteration 0: candidate of the initial bound set; if not optimal, start from
    // u = clip(uhat) (the clipped unconstrained maximiser when cold).
    pn_candidate<T, E, LPR>(y, u, bnd, w, l);
    bool ok = pn_test_direction<T, E, LPR, PE>(y, u, bnd, pin, w, lam, l);
    bool run = active && !ok;
    bool conv = active && ok, stall = false;
    if (run) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
            T lk = lam.at(k);
            if (!((bnd >> k) & 1u)) u[k] = clampv(u[k] + w[k], -lk, lk);
        }
    }
    int it = 1;        // candidate evaluations of this group's line
    int itw = 1;       // warp-uniform loop counter
    const int maxit = Num<T>::max_iters;
    while (itw < maxit && __any_sync(FULL, run)) {
        ++itw;
        uint32_t nb = pn_bound_set<T, E, LPR, PE>(y, u, pin, lam, l);
        if (run) bnd = nb;
        pn_candidate<T, E, LPR>(y, u, bnd, w, l);
        bool ok2 = pn_test_direction<T, E, LPR, PE>(y, u, bnd, pin, w, lam, l);
        if (run) it += 1;
        if (run && ok2) { conv = true; run = false; }
        bool ch = pn_line_search<T, E, LPR, PE>(y, u, w, bnd, lam, l, run);
        if (run && !ch) { stall = true; run = false; }
    }
    // output: the candidate of the final (u, B) when converged/stalled, else x(u)
    pn_candidate<T, E, LPR>(y, u, bnd, w, l);
    T uprev = shup<LPR>(u[E - 1], 1);
    if (l == 0) uprev = T(0);
    if (run) {
#pragma unroll
        for (int k = 0; k < E; ++k) w[k] = y[k] + u[k] - (k > 0 ? u[k > 0 ? k - 1 : 0] : uprev);
    }
    if (conv) return it;
    if (stall) return it | (1 << 16);
    return -1;
}

// ---------------------------------------------------------------------------
// Backward primitive: v <- segment-wise mean of v (Eq. 7 under reading O12:
// the symmetric projector onto vectors constant on the segments).  Segments end
// at edges in `bnd`; sgn(k) in {-1,0,+1} is the jump sign of edge k (pos/neg
// bitmasks).  lam_part += sum over segments ending in this lane of
// (s_R - s_L) * mean (dx/dlam = (s_R - s_L)/len).
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR>
__device__ __forceinline__ void seg_mean(T (&v)[E], uint32_t bnd, uint32_t pos, uint32_t neg, int l,
                                         T& lam_part) {
    T s = T(0);
    int c = 0;
    int sl = 0;       // sign of the edge before the open segment
    bool f = false;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        s += v[k];
        c += 1;
        if ((bnd >> k) & 1u) {
            f = true; s = T(0); c = 0;
            sl = ((pos >> k) & 1u) ? 1 : (((neg >> k) & 1u) ? -1 : 0);
        }
    }
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
        T s2 = shup<LPR>(s, d);
        int p2 = shup<LPR>(c | (f ? (1 << 30) : 0) | ((sl + 1) << 27), d);
        if (l >= d && !f) {
            s += s2; c += p2 & 0x7ffffff; f = (p2 >> 30) & 1; sl = ((p2 >> 27) & 3) - 1;
        }
    }
    T cs = shup<LPR>(s, 1);
    int cp = shup<LPR>(c | ((sl + 1) << 27), 1);
    if (l == 0) { cs = T(0); cp = (1 << 27); }
    s = cs; c = cp & 0x7ffffff; sl = ((cp >> 27) & 3) - 1;
    T first = T(0);
    bool hf = false;
    T lp = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k) {
        s += v[k];
        c += 1;
        if ((bnd >> k) & 1u) {
            T m = div_count(s, c);
            int sr = ((pos >> k) & 1u) ? 1 : (((neg >> k) & 1u) ? -1 : 0);
            lp += T(sr - sl) * m;
            v[k] = m;
            if (!hf) first = m;
            hf = true;
            sl = sr; s = T(0); c = 0;
        }
    }
    lam_part += lp;
    T vv = first;
    bool fv = hf;
#pragma unroll
    for (int d = 1; d < LPR; d <<= 1) {
        T v2 = shdn<LPR>(vv, d);
        int f2 = shdn<LPR>((int)fv, d);
        if (l + d < LPR && !fv) { vv = v2; fv = f2 != 0; }
    }
    T cur = shdn<LPR>(vv, 1);
#pragma unroll
    for (int k = E - 1; k >= 0; --k) {
        if ((bnd >> k) & 1u) cur = v[k]; else v[k] = cur;
    }
}

}  // namespace tvp
