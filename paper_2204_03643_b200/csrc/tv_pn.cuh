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
//
// One PN iteration is four fused lane passes over the E register-resident
// samples (P1 bound set + segment numerators, P2 carry + division, P3 reverse
// broadcast, P4 KKT test + uhat) and three warp scans; the Armijo line search
// only runs when the full step would leave the box.
#pragma once
#include "tv_common.cuh"
#include "tv_comm.cuh"
#ifdef TVP_DEBUG
#include <cstdio>
#endif

namespace tvp {


// Per-lane view of lambda: one value per line, or one per edge held in registers.
template <typename T, int E, bool PE>
struct Lam {
    T r;
    T e[PE ? E : 1];
    __device__ __forceinline__ T at(int k) const { return PE ? e[PE ? k : 0] : r; }
};

template <int E> __device__ __forceinline__ bool bit(uint32_t m, int k) { return (m & (1u << k)) != 0u; }

// Predicated accumulate / move (dst only changes where bit b of m is set): keeps the
// per-sample selects off the ALU pipe (predicated FADD / move instead of FSEL).
__device__ __forceinline__ void padd2(uint32_t m, uint32_t b, float& a0, float x0, float& a1, float x1) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "and.b32 t, %2, %3;\n\t"
        "setp.ne.u32 p, t, 0;\n\t"
        "@p add.f32 %0, %0, %4;\n\t"
        "@p add.f32 %1, %1, %5;\n\t}"
        : "+f"(a0), "+f"(a1) : "r"(m), "r"(b), "f"(x0), "f"(x1));
}
__device__ __forceinline__ void padd2(uint32_t m, uint32_t b, double& a0, double x0, double& a1, double x1) {
    if (m & b) { a0 += x0; a1 += x1; }
}

// Predicated-move forms of the P3 broadcast and the P4 running-sum restarts, per
// register geometry from same-box A/B runs: P4 wins except for
// the E = 14 half-warp lines (C5), P3 only for one-warp E = 16 lines (C4).
// TVP_P3_PTX / TVP_P4_PTX = 0 | 1 force them off / on everywhere.
template <int E, int LPR, int WPL> constexpr bool p3_ptx() {
#ifdef TVP_P3_PTX
    return TVP_P3_PTX != 0;
#else
    return E == 16 && LPR == 32 && WPL == 1;
#endif
}
template <int E, int LPR, int WPL> constexpr bool p4_ptx() {
#ifdef TVP_P4_PTX
    return TVP_P4_PTX != 0;
#else
    return E != 14;
#endif
}
// Largest E for which the segment pass uses the predicated-move form below (same-box
// A/B: it wins for the short 2D lines, E = 7, and loses for the two-warp E = 16 and the coarse
// E = 2 lines, where the compiler's own select scheduling is better).
#ifndef TVP_SEG_PTX_MAXE
#define TVP_SEG_PTX_MAXE 8
#endif
// ... and beyond it for the E = 14 half-warp lines (C5: fwd -4 %) and one-warp E = 16
// lines (C4: -2.5 %), same-box A/B (TVP_SEG_PTX_ALL=1 forces it for every E >= 4).
template <int E, int WPL> constexpr bool seg_ptx() {
#ifdef TVP_SEG_PTX_ALL
    return E >= 4;
#else
    return E >= 4 && (E <= TVP_SEG_PTX_MAXE || E == 14 || (E == 16 && WPL == 1));
#endif
}
// One sample of the lane-local segment pass (P1b) with predicated moves: w = num / cnt is
// written at every sample but read only where the edge is bound (the value of the segment
// ending there; the lane's first segment, which still lacks its carry, takes fv instead);
// numf keeps num at the lane's first bound edge; on a bound edge the running sums restart.
__device__ __forceinline__ void seg_step(uint32_t nb, uint32_t fbm, uint32_t b, float num, float cnt, float uk,
                                         float& w, float& numf, float& s, float& c) {
    asm("{\n\t.reg .pred pb, pf;\n\t.reg .b32 t1, t2;\n\t.reg .f32 r;\n\t"
        "and.b32 t1, %4, %6;\n\t"
        "setp.ne.u32 pb, t1, 0;\n\t"
        "and.b32 t2, %5, %6;\n\t"
        "setp.ne.u32 pf, t2, 0;\n\t"
        "rcp.approx.ftz.f32 r, %8;\n\t"
        "mul.f32 %0, %7, r;\n\t"
        "@pf mov.f32 %1, %7;\n\t"
        "@pb neg.f32 %2, %9;\n\t"
        "@pb mov.f32 %3, 0f00000000;\n\t}"
        : "+f"(w), "+f"(numf), "+f"(s), "+f"(c)
        : "r"(nb), "r"(fbm), "r"(b), "f"(num), "f"(cnt), "f"(uk));
}
__device__ __forceinline__ void seg_step(uint32_t nb, uint32_t fbm, uint32_t b, double num, double cnt, double uk,
                                         double& w, double& numf, double& s, double& c) {
    const bool bk = (nb & b) != 0u, fk = (fbm & b) != 0u;
    numf = fk ? num : numf;
    w = num * rcp_(cnt);
    s = bk ? -uk : s;
    c = bk ? 0.0 : c;
}

// Backward segment-mean steps in predicated form (float), see seg_mean_c.
__device__ __forceinline__ void segm1_step(uint32_t bnd, uint32_t fbm, uint32_t b, float s, float cnt,
                                           float& v, float& sf, float& so, float& co) {
    asm("{\n\t.reg .pred pb, pf;\n\t.reg .b32 t1, t2;\n\t.reg .f32 r;\n\t"
        "and.b32 t1, %4, %6;\n\t"
        "setp.ne.u32 pb, t1, 0;\n\t"
        "and.b32 t2, %5, %6;\n\t"
        "setp.ne.u32 pf, t2, 0;\n\t"
        "rcp.approx.ftz.f32 r, %8;\n\t"
        "@pf mov.f32 %1, %7;\n\t"
        "@pb mul.f32 %0, %7, r;\n\t"
        "mov.f32 %2, %7;\n\t"
        "mov.f32 %3, %8;\n\t"
        "@pb mov.f32 %2, 0f00000000;\n\t"
        "@pb mov.f32 %3, 0f00000000;\n\t}"
        : "+f"(v), "+f"(sf), "=f"(so), "=f"(co)
        : "r"(bnd), "r"(fbm), "r"(b), "f"(s), "f"(cnt));
}
__device__ __forceinline__ void segm1_step(uint32_t bnd, uint32_t fbm, uint32_t b, double s, double cnt,
                                           double& v, double& sf, double& so, double& co) {
    const bool bk = (bnd & b) != 0u, fk = (fbm & b) != 0u;
    sf = fk ? s : sf;
    v = bk ? s * rcp_(cnt) : v;
    so = bk ? 0.0 : s;
    co = bk ? 0.0 : cnt;
}
__device__ __forceinline__ void segm3_step(uint32_t bnd, uint32_t fm, uint32_t ng, uint32_t zs, uint32_t b, float fv,
                                           float& v, float& cur, float& sd, float& sn, float& sz) {
    asm("{\n\t.reg .pred pb, pf, pn, pz;\n\t.reg .b32 t1, t2, t3, t4;\n\t.reg .f32 x, d;\n\t"
        "and.b32 t1, %5, %9;\n\t"
        "setp.ne.u32 pb, t1, 0;\n\t"
        "and.b32 t2, %6, %9;\n\t"
        "setp.ne.u32 pf, t2, 0;\n\t"
        "and.b32 t3, %7, %9;\n\t"
        "setp.ne.u32 pn, t3, 0;\n\t"
        "and.b32 t4, %8, %9;\n\t"
        "setp.ne.u32 pz, t4, 0;\n\t"
        "mov.f32 x, %1;\n\t"
        "@pb mov.f32 x, %0;\n\t"
        "@pf mov.f32 x, %10;\n\t"
        "sub.f32 d, x, %1;\n\t"
        "add.f32 %2, %2, d;\n\t"
        "@pn add.f32 %3, %3, d;\n\t"
        "@pz add.f32 %4, %4, d;\n\t"
        "mov.f32 %0, x;\n\t"
        "mov.f32 %1, x;\n\t}"
        : "+f"(v), "+f"(cur), "+f"(sd), "+f"(sn), "+f"(sz)
        : "r"(bnd), "r"(fm), "r"(ng), "r"(zs), "r"(b), "f"(fv));
}
__device__ __forceinline__ void segm3_step(uint32_t bnd, uint32_t fm, uint32_t ng, uint32_t zs, uint32_t b, double fv,
                                           double& v, double& cur, double& sd, double& sn, double& sz) {
    double x = (bnd & b) ? v : cur;
    x = (fm & b) ? fv : x;
    const double d = x - cur;
    sd += d;
    sn += (ng & b) ? d : 0.0;
    sz += (zs & b) ? d : 0.0;
    v = x;
    cur = x;
}

// P3 reverse-broadcast step with predicated moves (the ALU pipe binds the forward;
// a predicated move issues on the FMA pipe, a select on the ALU pipe): off the bound
// edges the sample takes the running segment value, up to the lane's first bound it
// takes the carried first-segment value.
__device__ __forceinline__ void p3_step(uint32_t bnd, uint32_t firstm, uint32_t b, float fv, float& wk, float cur) {
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t1, t2;\n\t"
        "and.b32 t1, %1, %3;\n\t"
        "setp.eq.u32 p, t1, 0;\n\t"
        "and.b32 t2, %2, %3;\n\t"
        "setp.ne.u32 q, t2, 0;\n\t"
        "@p mov.f32 %0, %5;\n\t"
        "@q mov.f32 %0, %4;\n\t}"
        : "+f"(wk) : "r"(bnd), "r"(firstm), "r"(b), "f"(fv), "f"(cur));
}
__device__ __forceinline__ void p3_step(uint32_t bnd, uint32_t firstm, uint32_t b, double fv, double& wk, double cur) {
    double v = (bnd & b) ? wk : cur;
    wk = (firstm & b) ? fv : v;
}
// P4 running sums restarted at bound edges: r = u_k, A = |u_k| there (predicated moves).
__device__ __forceinline__ void p4_restart(uint32_t bnd, uint32_t b, float uk, float t, float& r, float& A) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t1;\n\t.reg .f32 at;\n\t"
        "and.b32 t1, %2, %3;\n\t"
        "setp.ne.u32 p, t1, 0;\n\t"
        "add.f32 %0, %0, %5;\n\t"
        "abs.f32 at, %5;\n\t"
        "add.f32 %1, %1, at;\n\t"
        "@p mov.f32 %0, %4;\n\t"
        "@p abs.f32 %1, %4;\n\t}"
        : "+f"(r), "+f"(A) : "r"(bnd), "r"(b), "f"(uk), "f"(t));
}
__device__ __forceinline__ void p4_restart(uint32_t bnd, uint32_t b, double uk, double t, double& r, double& A) {
    const bool bk = (bnd & b) != 0u;
    r = bk ? uk : r + t;
    A = bk ? fabs(uk) : A + fabs(t);
}

// Selects of the reverse P3/P4 pass: xhat_k = fv on the lane's first segment (bits 0..fb),
// else the segment value w_k on a bound edge, else xhat_{k+1}; uhat_k = u_k restarts on a
// bound edge, else the value carried from edge k + 1.
__device__ __forceinline__ void p34_sel(uint32_t bnd, uint32_t firstm, uint32_t b, float fv, float wk, float xr,
                                        float uk, float rr, float& xh, float& r) {
    // (results built in asm-local registers: "=f" outputs may share a register with an input)
    asm("{\n\t.reg .pred pb, pf;\n\t.reg .b32 t1, t2;\n\t.reg .f32 x, rv;\n\t"
        "and.b32 t1, %2, %4;\n\t"
        "setp.ne.u32 pb, t1, 0;\n\t"
        "and.b32 t2, %3, %4;\n\t"
        "setp.ne.u32 pf, t2, 0;\n\t"
        "mov.f32 x, %7;\n\t"
        "@pb mov.f32 x, %6;\n\t"
        "@pf mov.f32 x, %5;\n\t"
        "mov.f32 rv, %9;\n\t"
        "@pb mov.f32 rv, %8;\n\t"
        "mov.f32 %0, x;\n\t"
        "mov.f32 %1, rv;\n\t}"
        : "=f"(xh), "=f"(r)
        : "r"(bnd), "r"(firstm), "r"(b), "f"(fv), "f"(wk), "f"(xr), "f"(uk), "f"(rr));
}
__device__ __forceinline__ void p34_sel(uint32_t bnd, uint32_t firstm, uint32_t b, double fv, double wk, double xr,
                                        double uk, double rr, double& xh, double& r) {
    const bool bk = (bnd & b) != 0u;
    xh = (firstm & b) ? fv : (bk ? wk : xr);
    r = bk ? uk : rr;
}

// m |= b  iff  ug > 0 and au >= thr, as two compares (the second predicated on the
// first) and one predicated OR -- the ALU pipe is the forward's binding pipe.
__device__ __forceinline__ void or_if_outward(uint32_t& m, float ug, float au, float thr, uint32_t b) {
    asm("{\n\t.reg .pred p, q;\n\t"
        "setp.gt.f32 p, %1, 0f00000000;\n\t"
        "setp.ge.and.f32 q, %2, %3, p;\n\t"
        "@q or.b32 %0, %0, %4;\n\t}"
        : "+r"(m) : "f"(ug), "f"(au), "f"(thr), "r"(b));
}
__device__ __forceinline__ void or_if_outward(uint32_t& m, double ug, double au, double thr, uint32_t b) {
    asm("{\n\t.reg .pred p, q;\n\t"
        "setp.gt.f64 p, %1, 0d0000000000000000;\n\t"
        "setp.ge.and.f64 q, %2, %3, p;\n\t"
        "@q or.b32 %0, %0, %4;\n\t}"
        : "+r"(m) : "d"(ug), "d"(au), "d"(thr), "r"(b));
}

// Highest set bit of m below position k, or -1.
__device__ __forceinline__ int prev_bit(uint32_t m, int k) {
    uint32_t mm = k >= 32 ? m : (m & ((1u << k) - 1u));
    return 31 - __clz(mm);
}

// Line-search configuration (DESIGN.md a-7, f3).  From PN iteration ls_after on (a runtime
// argument, tvp_options_t.ls_after; default kLsAfterDefault), a step whose full Newton
// point leaves the box is globalised by the projected Armijo line search of P:188;
// before that it is the projected full step.  The search flavour is a template
// parameter LSP of the solver (separate kernel instantiations, so the default kernels
// carry no code of the other flavour): false = sequential quadratic-interpolation
// backtracking ("only iterates a few times"), true = the parallel step search
// (SURVEY 8(f) f3): four step sizes alpha, alpha/2, alpha/4, alpha/8 evaluated in one
// fused pass with one reduction, the largest Armijo-accepted one taken.
constexpr int kLsAfterDefault = 12;

template <typename T> __device__ __forceinline__ T big_();
template <> __device__ __forceinline__ float big_<float>() { return 3.0e38f; }
template <> __device__ __forceinline__ double big_<double>() { return 1.0e300; }

// ---------------------------------------------------------------------------
// The solver.  y: centred samples (read-only); u: dual (in/out); w: output x
// (centred).  pin: pinned edges.  warm_pos/warm_neg: edges that were up/down
// jumps in a previous solve (warm start, DESIGN.md a-11).  lam_max: max lambda
// of the line (slack bound).  Returns the line status: iterations (| 1<<16 if
// accepted at a stall), or -1 (max iterations, w = x(u)).
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR, int WPL, bool PE, bool LSP = false, typename CM = Comm<T, LPR, WPL>>
__device__ __forceinline__ int pn_solve(const T (&y)[E], T (&u)[E], T (&w)[E], uint32_t pin,
                                        uint32_t warm_pos, uint32_t warm_neg,
                                        const Lam<T, E, PE>& lam, const CM& C,
                                        bool active, int ls_after, int& ls_passes, int max_iters = 0) {
    warm_pos &= ~pin;
    warm_neg &= ~pin;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const T lk = lam.at(k);
        u[k] = bit<E>(warm_pos, k) ? lk : (bit<E>(warm_neg, k) ? -lk : T(0));
    }
    uint32_t bnd = pin | warm_pos | warm_neg;
    uint32_t bnd2 = 0xffffffffu;       // bound set two iterations ago (cycle detection)
    uint32_t bnd3 = 0xffffffffu, bnd4 = 0xffffffffu;   // three / four ago (cluster lines only)
    const T ynext = C.template next<1>(y[0]);
    // lane constants of the reverse uhat carry (P3/P4): sum of |y| over the lane's samples
    // and the largest lambda of the lane
    T yabs = T(0), lmaxl = lam.at(0);
#pragma unroll
    for (int k = 0; k < E; ++k) {
        yabs += fabs(y[k]);
        if (PE) lmaxl = fmax(lmaxl, lam.at(k));
    }
    const T eps = Num<T>::eps;
    const T slackA = eps * T(8);     // summation-error slack of the KKT test (x sum |terms|)
    const T slack1 = T(1) + T(2) * eps;
    const int maxit = max_iters > 0 ? max_iters : Num<T>::max_iters;

    // Line state.  Only run / fin / uchg are bools across the loop, the exit kind is an int
    // and `first` is itw == 0: the per-sample loops need the predicate registers (with more
    // long-lived bools the compiler packs predicates into a register, two LOP3 per save /
    // restore, inside those loops).  Same-box A/B: C2 fwd 1.207 -> 1.133 ms, C5 4.08 -> 3.94;
    // turning fin / uchg (and solve_line's active / bad) into ints as well measured slower.
    bool run = active, fin = false, uchg = true;
    int how = 0;                       // 1: converged, 2: accepted at a stall
    int it = 0;
    ls_passes = 0;
    for (int itw = 0;; ++itw) {
        const bool first = itw == 0;
        // ---------------- P1: bound set at u (Bertsekas rule: at a bound with the
        // gradient g = D x(u) pointing out of the box) fused with the lane-local part
        // of the Eq. 6 partition solve: each segment ending in the lane gets
        //   xhat = (sum_y - u_{a-1} + u_{b-1}) / len ;  s carries sum_y - u_{a-1}.
        const bool upd = run && !first && !fin;
        const uint32_t keep = upd ? pin : bnd;
        T uprev = T(0), unext = T(0);
        // (a) outward-gradient bits at the bound (predicate -> one OR per sample); not
        // needed when no line of the warp updates its bound set (the first step from
        // the initial set, the final candidate pass): outb would be 0 there
        uint32_t outb = 0;
        if (C.uany(upd)) {
            C.template prev_next<0>(u[E - 1], u[0], uprev, unext);
            T xk = y[0] + u[0] - uprev;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const T thr = upd ? lam.at(k) : big_<T>();
                const T xk1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                                          : (ynext + unext - u[k]);
                const T g = xk1 - xk;
                xk = xk1;
                or_if_outward(outb, u[k] * g, fabs(u[k]), thr, 1u << k);
            }
        }
        const uint32_t nb = keep | outb;
        const uint32_t firstb = nb & (0u - nb);         // lowest bound edge of the lane
        // (b) lane-local segment numerators / values with the final bits
        T s = T(0), cnt = T(0), numf = T(0);
#pragma unroll
        for (int k = 0; k < E; ++k) {
            s += y[k];
            cnt += T(1);
            const T num = s + u[k];
            if constexpr (seg_ptx<E, WPL>()) {
                seg_step(nb, firstb, 1u << k, num, cnt, u[k], w[k], numf, s, cnt);
            } else {
                const bool bk = bit<E>(nb, k);
                const bool fk = bit<E>(firstb, k);
                numf = fk ? num : numf;
                w[k] = num * rcp_(cnt);            // read only where edge k is bound (after P1b)
                s = bk ? -u[k] : s;
                cnt = bk ? T(0) : cnt;
            }
        }
        const bool bchg = C.any(nb != bnd);
        // rounding-level fixed point (no change) or 2-cycle of the bound set: stall
        bool cyc2;
        if constexpr (CM::kCluster) {
            // lines of 10^4..10^5 samples (f4) can cycle through bound sets with period 2..4
            // under projected full Newton steps in fp32; one vote covers the three periods.
            // A cycle switches the line to the Armijo-globalised step for the
            // rest of the solve, whose accepted steps strictly increase the dual objective;
            // only a cycle under the line search is a rounding-level stall (O7).
            const uint32_t eq = (nb == bnd2 ? 1u : 0u) | (nb == bnd3 ? 2u : 0u) | (nb == bnd4 ? 4u : 0u);
            cyc2 = bchg & (C.all_bits(eq) != 0u);
            bnd4 = bnd3;
            bnd3 = bnd2;
            if (cyc2 && it + 1 < ls_after) {
                ls_after = it + 1;
                cyc2 = false;
            }
        } else {
            if constexpr (WPL > 1) {
                // lines of several warps: the vote is a block barrier; skip it before a set from
                // two iterations ago exists and while the set is unchanged (block-uniform
                // conditions).  C2 fwd 1.093 -> 1.049 ms; for warp-level votes the extra
                // uniformity test costs more than the ballot it saves (C5 +2 %).
                cyc2 = (itw >= 2 && bchg) ? C.all(nb == bnd2) : false;
            } else {
                cyc2 = bchg & C.all(nb == bnd2);
            }
        }
        if (upd && ((!uchg && !bchg) || cyc2)) { how = 2; run = false; }
        bnd2 = bnd;
        bnd = nb;
        const int hb = 31 - __clz(bnd);              // -1 if none
        const bool fl = bnd != 0u;
        const int cnt_tail = E - 1 - hb;
        const auto sg = C.seg_plan(fl);               // segment geometry of this step's scans

        // ---------------- P2: the lane's first segment gets the carry.
        const int fb = __ffs(bnd) - 1;                // -1 if none
        const uint32_t firstm = bnd ? ((bnd & (0u - bnd)) * 2u - 1u) : 0u;   // bits 0..fb
        // Then the value of the segment that runs into this lane from the right (cur): the
        // first-segment value fv of the nearest flagged line lane to the right.  It is also
        // xhat of the next line lane's first sample (that lane's fv if it is flagged, else the
        // value it receives from the same source), so no neighbour exchange is needed for it.
        // And the lane aggregates of the reverse uhat carry (P3/P4 below).  Two-warp lines do
        // all three scans in one block exchange (Comm::scan_all2: the carry is rebuilt from
        // cur-independent sums over the flagless lanes, rr = Vh + S - E N cur); other lines
        // add the flagless lanes' value-dependent parts after cur arrives.
        constexpr bool kRevC = !CM::kCluster && WPL == 2;
        T fv, rr, AA, cur;
        if constexpr (kRevC) {
            C.template scan_all2<2, E>(sg, fl, s, cnt_tail, numf, fb, lmaxl, yabs, fv, rr, AA, cur);
        } else {
            T cs = s;
            int cc = cnt_tail;
            C.template scan_fwd<2, E>(sg, cs, cc);
            fv = (numf + cs) * rcp_(T(fb + 1 + cc));
            rr = fl ? (numf - T(fb + 1) * fv) : s;
            AA = fl ? (lmaxl + T(fb + 1) * fabs(fv)) + yabs : yabs;
            cur = C.template scan_rev<3>(sg, fv);
        }
        bool ok = true, clip = false, chg = false;
        bool lsmode;
        if constexpr (CM::kCluster) {
            // Lines held by a thread-block cluster (f4) keep the forward form of P3/P4: a
            // reverse broadcast pass that also sums xhat - y over the lane's open tail, a
            // forward segmented scan of (uhat, slack scale) from each segment's left end, and
            // a forward KKT / step pass -- with explicit change detection for the stall rule
            // (their cycle handling switches lines to the Armijo step, see above).
            const uint32_t tailm = fl ? ~((2u << hb) - 1u) : 0xffffffffu;
            T rt = T(0), at = T(0), ub = T(0);
#pragma unroll
            for (int k = 0; k < E; ++k) ub = bit<E>(bnd, k) ? u[k] : ub;     // u at the lane's last bound edge
            const T xnext = cur;
#pragma unroll
            for (int k = E - 1; k >= 0; --k) {
                T v = bit<E>(bnd, k) ? w[k] : cur;
                v = bit<E>(firstm, k) ? fv : v;
                w[k] = v;
                cur = v;
                const T t = v - y[k];
                padd2(tailm, 1u << k, rt, t, at, fabs(t));
            }
            if (fin) break;
            T r = ub + rt;
            T A = fabs(ub) + at;
            C.template scan_fwd2<4>(sg, r, A);
            lsmode = C.uany(run && !first && (it + 1 >= ls_after));
            if (!lsmode) {
                T vio = T(0), dch = T(0);
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const T xh = w[k];
                    const T xh1 = (k + 1 < E) ? w[(k + 1 < E) ? k + 1 : k] : xnext;
                    const T t = xh - y[k];
                    const T lk = lam.at(k);
                    p4_restart(bnd, 1u << k, u[k], t, r, A);
                    const T q = u[k] * (xh1 - xh);
                    const T e = fabs(r) - fma(slackA, AA, lk * slack1);
                    vio += (fabs(q) - q) + (e + fabs(e));
                    dch += fabs(r - u[k]);
                    u[k] = clampv(r, -lk, lk);
                }
                ok = vio == T(0);
                chg = dch != T(0);
            } else {
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const T xh = w[k];
                    const T xh1 = (k + 1 < E) ? w[(k + 1 < E) ? k + 1 : k] : xnext;
                    const T t = xh - y[k];
                    r += t;
                    A += fabs(t);
                    const T lk = lam.at(k);
                    const bool bk = bit<E>(bnd, k);
                    const bool sgn_bad = u[k] * (xh1 - xh) < T(0);      // pinned edges: u = 0
                    const T ar = fabs(r);
                    const bool infeas = ar > fma(slackA, A, lk * slack1);
                    ok = ok & !(bk ? sgn_bad : infeas);
                    clip = clip | (!bk & (ar > lk));
                    chg = chg | (!bk & (r != u[k]));
                    w[k] = bk ? u[k] : r;
                    A = bk ? fabs(u[k]) : A;
                    r = bk ? u[k] : r;
                }
                clip = C.any(clip);
            }
            chg = C.any(chg);
        } else {
            if (fin) {
                // final candidate pass: reverse broadcast of each segment's value to its samples
#pragma unroll
                for (int k = E - 1; k >= 0; --k) {
                    T v;
                    if constexpr (p3_ptx<E, LPR, WPL>()) {
                        p3_step(bnd, firstm, 1u << k, fv, w[k], cur);
                        v = w[k];
                    } else {
                        v = bit<E>(bnd, k) ? w[k] : cur;
                        v = bit<E>(firstm, k) ? fv : v;
                        w[k] = v;
                    }
                    cur = v;
                }
                break;
            }

            // ---------------- P3/P4 (one reverse pass): broadcast of the segment values, KKT /
            // zero-duality-gap test of the candidate, and the dual uhat computed from each
            // segment's right end:  uhat_{b-1} = u_{b-1} on a bound edge b-1 and, on a free edge,
            //     uhat_i = uhat_{i+1} - (xhat_{i+1} - y_{i+1})
            // (the same uhat as the running sum from the left end, since the partition value
            // makes each segment's sum of xhat - y equal u_{b-1} - u_{a-1}).  Free edges must
            // satisfy |uhat_i| <= lam_i (up to a summation-error slack), bound edges must jump in
            // the direction of u_i.  Fast mode (no line search possible this iteration) applies
            // the projected full Newton step u <- clip(uhat) in the same pass and keeps xhat in w;
            // LS mode writes uhat to w for the search.
            // The carry into the lane's last edge is a reverse segmented scan of the lanes' sums
            // of -(xhat - y), O(1) per lane: a flagged lane's head [0, fb] sums to
            // -((fb+1) fv - (numf - u_fb)) = numf - (fb+1) fv - u_fb, so it hands u_fb - that =
            // numf - (fb+1) fv to its left; a flagless lane sums to E cur - s (s = its sample sum
            // from P1b).  The slack scale carried with it is an upper bound of the matching
            // |u| + sum |xhat - y| (|xhat - y_j| <= |xhat| + |y_j|); inside the lane it keeps
            // accumulating |xhat - y| across bound edges (no restart: a larger, still valid
            // bound on free edges; on bound edges |uhat| = |u| <= lam never reads it).
            if constexpr (!kRevC) {
                if (!fl) {
                    rr -= T(E) * cur;
                    AA += T(E) * fabs(cur);
                }
                C.template scan_rev2<4>(sg, rr, AA);
            }
            lsmode = C.uany(run && !first && (it + 1 >= ls_after));
            T xr = cur;                                   // xhat_{k+1}
            if (!lsmode) {
                // The tests accumulate non-negative violations on the FMA pipe instead of
                // predicate logic (the ALU pipe binds this loop):
                //  * r, A restart at bound edges (r = u_i there, so |r| <= lam_i never
                //    reads as infeasible and clamp(r) = u_i keeps the bound value);
                //  * sign test u_i (xhat_{i+1} - xhat_i) >= 0 needs no bound mask: across a
                //    free edge both samples carry the same segment value bitwise (product 0),
                //    and pinned edges have u = 0;
                //  * |q| - q > 0 iff q < 0 and e + |e| > 0 iff e > 0, exactly (no FTZ), and
                //    a sum of non-negative terms is 0 iff every term is.
                T vio = T(0);
#pragma unroll
                for (int k = E - 1; k >= 0; --k) {
                    T xh, r;
                    p34_sel(bnd, firstm, 1u << k, fv, w[k], xr, u[k], rr, xh, r);
                    const T lk = lam.at(k);
                    const T q = u[k] * (xr - xh);
                    const T e = fabs(r) - fma(slackA, AA, lk * slack1);
                    vio += (fabs(q) - q) + (e + fabs(e));
                    const T t = xh - y[k];
                    rr = r - t;
                    AA += fabs(t);
                    u[k] = clampv(r, -lk, lk);
                    w[k] = xh;
                    xr = xh;
                }
                ok = vio == T(0);
            } else {
#pragma unroll
                for (int k = E - 1; k >= 0; --k) {
                    T xh, r;
                    p34_sel(bnd, firstm, 1u << k, fv, w[k], xr, u[k], rr, xh, r);
                    const T lk = lam.at(k);
                    const bool bk = bit<E>(bnd, k);
                    const bool sgn_bad = u[k] * (xr - xh) < T(0);      // pinned edges: u = 0
                    const T ar = fabs(r);
                    const bool infeas = ar > fma(slackA, AA, lk * slack1);
                    ok = ok & !(bk ? sgn_bad : infeas);
                    clip = clip | (!bk & (ar > lk));
                    const T t = xh - y[k];
                    rr = r - t;
                    AA += fabs(t);
                    w[k] = r;                             // uhat (u_k on bound edges)
                    xr = xh;
                }
                clip = C.any(clip);
            }
        }
        ok = C.all(ok);
#ifdef TVP_DEBUG
        if (active && C.first_lane())
            printf("[tvp] itw %d it %d run %d first %d ok %d clip %d bchg %d uchg %d nbound %d ls %d\n", itw, it,
                   (int)run, (int)first, (int)ok, (int)clip, (int)bchg, (int)uchg, __popc(bnd), (int)lsmode);
#endif
        if (run) ++it;
        if (run && ok) { how = 1; run = false; }
        // every line of the warp has stopped after a fast-mode step: this step's P3 left
        // each line's candidate in w (a line that stopped earlier recomputes the same
        // candidate bitwise: its bound set is frozen and xhat reads u only on bound
        // edges), so the final candidate pass is not needed
        if (!lsmode && !C.uany(run)) break;

        // ---------------- step (LS mode): full Newton step when it stays in the box,
        // else the projected Armijo line search with quadratic-interpolation
        // backtracking of P:188 -- the globalisation safeguard from iteration ls_after on.
        // After a full (projected) Newton step the next candidate depends only on the next
        // bound set (xhat reads u on bound edges, which keep their values), so a bound set
        // equal to this one reproduces this failed candidate bitwise: the step is a
        // rounding-level fixed point, detected by bchg alone (uchg = false).  Only an
        // Armijo step (below) changes u without changing the candidate.
        const bool fast = lsmode && run && (first || !clip);
        if (!lsmode) {
            uchg = (CM::kCluster && chg) || first;
        } else if (fast) {
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const T lk = lam.at(k);
                u[k] = bit<E>(bnd, k) ? u[k] : clampv(w[k], -lk, lk);
            }
            uchg = (CM::kCluster && chg) || first;
        }
        bool pending = lsmode && run && !fast;
        if (LSP && C.uany(pending)) {
            constexpr int NA = 4;
            T abase = T(1), alpha = T(0);
            bool accepted = false, lchg = false;
            for (int round = 0; round < 8; ++round) {
                if (!C.uany(pending)) break;
                const T lkl = lam.at(E - 1);
                T dprev[NA];
#pragma unroll
                for (int j = 0; j < NA; ++j) {
                    const T aj = abase * T(1.0 / (1 << j));
                    const T dlast = bit<E>(bnd, E - 1) ? T(0)
                                                       : clampv(u[E - 1] + aj * (w[E - 1] - u[E - 1]), -lkl, lkl) - u[E - 1];
                    dprev[j] = (j == 0) ? C.template prev<12>(dlast)
                             : (j == 1) ? C.template prev<13>(dlast)
                             : (j == 2) ? C.template prev<14>(dlast) : C.template prev<15>(dlast);
                }
                T F[NA], Gs[NA];
                bool ch[NA];
#pragma unroll
                for (int j = 0; j < NA; ++j) { F[j] = T(0); Gs[j] = T(0); ch[j] = false; }
                T x0 = y[0] + u[0] - uprev;
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const T lk = lam.at(k);
                    const T dk = bit<E>(bnd, k) ? T(0) : (w[k] - u[k]);
                    const T x1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                                             : (ynext + unext - u[k]);
                    const T g = x1 - x0;
#pragma unroll
                    for (int j = 0; j < NA; ++j) {
                        const T aj = abase * T(1.0 / (1 << j));
                        const T du = clampv(u[k] + aj * dk, -lk, lk) - u[k];
                        const T dl = du - dprev[j];
                        F[j] = fma(dl, T(2) * x0 + dl, F[j]);
                        Gs[j] = fma(g, du, Gs[j]);
                        ch[j] = ch[j] | (du != T(0));
                        dprev[j] = du;
                    }
                    x0 = x1;
                }
                T z = T(0);
                C.template sum3<7>(F[0], F[1], F[2]);
                C.template sum3<9>(F[3], Gs[0], Gs[1]);
                C.template sum3<11>(Gs[2], Gs[3], z);
                bool chj[NA];
#pragma unroll
                for (int j = 0; j < NA; ++j) chj[j] = C.any(ch[j]);
                if (pending) {
                    ++ls_passes;
#pragma unroll
                    for (int j = NA - 1; j >= 0; --j) {     // keep the largest accepted alpha
                        const T gain = T(-0.5) * F[j];
                        if (gain >= T(1e-4) * Gs[j]) {
                            alpha = abase * T(1.0 / (1 << j));
                            accepted = gain > T(0);
                            lchg = chj[j];
                        }
                    }
                    if (alpha > T(0)) pending = false;
                    abase *= T(1.0 / (1 << NA));
                    if (abase < T(1e-12)) pending = false;
                }
            }
            if (lsmode && run && !fast) {
                if (accepted && lchg) {
#pragma unroll
                    for (int k = 0; k < E; ++k) {
                        const T lk = lam.at(k);
                        const T dk = bit<E>(bnd, k) ? T(0) : (w[k] - u[k]);
                        u[k] = clampv(u[k] + alpha * dk, -lk, lk);
                    }
                    uchg = true;
                } else {
                    how = 2;
                    run = false;
                }
            }
        } else if (C.uany(pending)) {
            T alpha = T(1), slope = T(0);
            bool accepted = false, lchg = false;
            for (int trial = 0; trial < 30; ++trial) {
                if (!C.uany(pending)) break;
                const T lkl = lam.at(E - 1);
                const T dlast = bit<E>(bnd, E - 1) ? T(0)
                                                   : clampv(u[E - 1] + alpha * (w[E - 1] - u[E - 1]), -lkl, lkl) - u[E - 1];
                T duprev = C.template prev<6>(dlast);
                T F = T(0), G = T(0), S = T(0);
                bool ch = false;
                T x0 = y[0] + u[0] - uprev;
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const T lk = lam.at(k);
                    const T dk = bit<E>(bnd, k) ? T(0) : (w[k] - u[k]);
                    const T du = clampv(u[k] + alpha * dk, -lk, lk) - u[k];
                    const T x1 = (k + 1 < E) ? (y[(k + 1 < E) ? k + 1 : k] + u[(k + 1 < E) ? k + 1 : k] - u[k])
                                             : (ynext + unext - u[k]);
                    const T g = x1 - x0;
                    const T dl = du - duprev;
                    F = fma(dl, T(2) * x0 + dl, F);
                    G = fma(g, du, G);
                    S = fma(g, dk, S);
                    ch = ch | (du != T(0));
                    duprev = du;
                    x0 = x1;
                }
                C.template sum3<7>(F, G, S);
                ch = C.any(ch);
                if (trial == 0) slope = S;
#ifdef TVP_DEBUG
                if (pending && C.first_lane()) printf("[tvp]   LS trial %d alpha %g F %g G %g S %g ch %d\n", trial, (double)alpha, (double)F, (double)G, (double)S, (int)ch);
#endif
                if (pending) {
                    ++ls_passes;
                    const T gain = T(-0.5) * F;          // phi(u(alpha)) - phi(u)
                    if (gain >= T(1e-4) * G) {
                        // an accepted step without measurable ascent is a rounding-level
                        // fixed point: stall (O8)
                        pending = false; accepted = gain > T(0); lchg = ch;
                    } else {
                        const T den = T(2) * (slope * alpha - gain);
                        const T an = den > T(0) ? slope * alpha * alpha / den : T(0.5) * alpha;
                        alpha = clampv(an, T(0.1) * alpha, T(0.5) * alpha);
                        if (alpha < T(1e-12)) pending = false;
                    }
                }
            }
            if (lsmode && run && !fast) {
                if (accepted && lchg) {
#pragma unroll
                    for (int k = 0; k < E; ++k) {
                        const T lk = lam.at(k);
                        const T dk = bit<E>(bnd, k) ? T(0) : (w[k] - u[k]);
                        u[k] = clampv(u[k] + alpha * dk, -lk, lk);
                    }
                    uchg = true;
                } else {
                    how = 2;                               // no ascent step exists at rounding level
                    run = false;
                }
            }
        }
        if (!C.uany(run) || itw + 2 >= maxit) fin = true;
    }
    // lines still running hit max_iters: output the primal of the current dual
    const T upv = C.template prev<10>(u[E - 1]);
    if (run) {
#pragma unroll
        for (int k = 0; k < E; ++k) w[k] = y[k] + u[k] - (k > 0 ? u[k > 0 ? k - 1 : 0] : upv);
        return -1;
    }
    if (how == 1) return it;
    if (how == 2) return it | (1 << 16);
    return 0;
}

// ---------------------------------------------------------------------------
// Coarse initial bound set for a cold solve (reading O7).  The line is
// cut into the lanes' blocks of E samples; restricting x to be constant on full
// blocks turns Eq. 1 into the same prox on the block means with lam / E:
//     1/2 sum_b E (x_b - ybar_b)^2 + lam sum_b |x_{b+1} - x_b|.
// That nc = n / E sample problem is solved by the same projected Newton method
// (pn_solve), and its jumps become the initial bound edges of the fine solve
// (u = +lam on an up jump, -lam on a down jump, at the block's last edge).  Only
// the PN iteration count depends on this; the fine solve's answer does not.
//   WPL == 1: coarse sample b is held by line lane b (one per lane, in place).
//   WPL  > 1: block means are exchanged through xb[32*WPL] (shared memory) and
//             every warp solves the whole coarse line redundantly (WPL samples
//             per lane, warp shuffles only); jump bits come back by ballots.
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR, int WPL, typename CM = Comm<T, LPR, WPL>>
__device__ __forceinline__ void coarse_init(const T (&y)[E], T lam_r, int n, bool active,
                                            const CM& C, T* xb,
                                            uint32_t& cpos, uint32_t& cneg) {
    const int ll = C.w * LPR + C.l;
    const int nc = n / E;
    T bs = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k) bs += y[k];
    const T ybar = (ll < nc) ? bs * (T(1) / T(E)) : T(0);
    Lam<T, WPL, false> lc;
    lc.r = lam_r * (T(1) / T(E));
    constexpr uint32_t top = 1u << (E - 1);
    cpos = cneg = 0u;
    if constexpr (WPL == 1) {
        T yc[WPL], uc[WPL], wc[WPL];
        yc[0] = ybar;
        const uint32_t pinc = (ll >= nc - 1) ? 1u : 0u;
        int lsp_;
        pn_solve<T, WPL, LPR, 1, false>(yc, uc, wc, pinc, 0u, 0u, lc, C, active, kLsAfterDefault, lsp_);
        const T xn = shdn<LPR>(wc[0], 1);
        if (ll < nc - 1) {
            cpos = xn > wc[0] ? top : 0u;
            cneg = xn < wc[0] ? top : 0u;
        }
    } else {
        xb[ll] = ybar;
        __syncthreads();
        const int l = C.l;
        T yc[WPL], uc[WPL], wc[WPL];
        uint32_t pinc = 0u;
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
            yc[q] = xb[l * WPL + q];
            pinc |= (l * WPL + q >= nc - 1) ? (1u << q) : 0u;
        }
        const Comm<T, 32, 1> Cw{l, 0, nullptr, nullptr};
        int lsp_;
        pn_solve<T, WPL, 32, 1, false>(yc, uc, wc, pinc, 0u, 0u, lc, Cw, active, kLsAfterDefault, lsp_);
        const T xn = shdn<32>(wc[0], 1);
        const int cl = ll / WPL, cq = ll % WPL;
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
            const T nx = (q + 1 < WPL) ? wc[(q + 1 < WPL) ? q + 1 : q] : xn;
            const bool inl = l * WPL + q < nc - 1;
            const uint32_t bu = __ballot_sync(FULL, inl && nx > wc[q]);
            const uint32_t bd = __ballot_sync(FULL, inl && nx < wc[q]);
            if (q == cq) {
                cpos = ((bu >> cl) & 1u) ? top : 0u;
                cneg = ((bd >> cl) & 1u) ? top : 0u;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Backward primitive: v <- segment-wise mean of v (Eq. 7 under reading O12:
// the symmetric projector onto vectors constant on the segments), for a line
// held by a Comm group.  Segments end at edges in `bnd`; the jump sign of edge
// k is +1 (pos), -1 (neg) or 0.  lam_part += sum_e s_e (mean_left(e) -
// mean_right(e)) = sum_seg (s_R - s_L) mean_seg (dx/dlam = (s_R - s_L)/len).
// Comm slots 0..2 are used.
// ---------------------------------------------------------------------------
template <typename T, int E, int LPR, int WPL, typename CM = Comm<T, LPR, WPL>>
__device__ __forceinline__ void seg_mean_c(T (&v)[E], uint32_t bnd, uint32_t pos, uint32_t neg,
                                           const CM& C, T& lam_part) {
    // pass 1: means of the segments that end inside the lane; the lane's first
    // segment keeps its partial sum (it still lacks the carry), the open tail sum
    // goes to the scan
    const uint32_t firstb = bnd & (0u - bnd);
    T s = T(0), sf = T(0), cnt = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k) {
        s += v[k];
        cnt += T(1);
        segm1_step(bnd, firstb, 1u << k, s, cnt, v[k], sf, s, cnt);
    }
    const int hb = 31 - __clz(bnd);
    const bool fl = bnd != 0u;
    T cs = s;
    int cc = E - 1 - hb;
    const auto sg = C.seg_plan(fl);
    C.template scan_fwd<0, E>(sg, cs, cc);
    const int fb = __ffs(bnd) - 1;
    const uint32_t firstm = bnd ? (firstb * 2u - 1u) : 0u;
    const T fv = (sf + cs) * rcp_(T(fb + 1 + cc));
    // pass 3 (reverse): broadcast each segment's mean to its samples, and the lambda
    // gradient in edge form, sum_e s_e (mean_L(e) - mean_R(e)): d = x_k - (value to
    // the right) is exactly 0 inside a segment, so sum_e s_e d_e = sum d - 2 sum_neg d
    // - sum_bnd d, the last term over edges coded "boundary" (s = 0: lam = 0, pinned).
    T cur = C.template scan_rev<2>(sg, fv);
    const uint32_t zs = bnd & ~(pos | neg);          // edges with zero sign
    T sd = T(0), sn = T(0), sz = T(0);
#pragma unroll
    for (int k = E - 1; k >= 0; --k) segm3_step(bnd, firstm, neg, zs, 1u << k, fv, v[k], cur, sd, sn, sz);
    const T lp = sd - T(2) * sn - sz;
    lam_part += lp;
}

// Warp-group form (WPL = 1) used by the tiled column / short-row kernels.
template <typename T, int E, int LPR>
__device__ __forceinline__ void seg_mean(T (&v)[E], uint32_t bnd, uint32_t pos, uint32_t neg, int l,
                                         T& lam_part) {
    const Comm<T, LPR, 1> C{l, 0, nullptr, nullptr};
    seg_mean_c<T, E, LPR, 1>(v, bnd, pos, neg, C, lam_part);
}

}  // namespace tvp
