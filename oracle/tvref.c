/*
 * oracle/tvref.c -- CPU ORACLE for arXiv 2204.03643 ("Total Variation
 * Optimization Layers for Computer Vision", Yeh, Hu, Ren, Schwing).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2204_03643_b200/, libtvprox.so) never links,
 * imports or calls it, and this file shares no code, header, table or
 * helper with the CUDA path.
 *
 * Plain, slow, obviously-correct fp64 (long double where noted) C99.
 * Notation follows the ABI / SURVEY.md section 0: input y, output x,
 *   x = argmin_x 1/2 ||x - y||^2 + lam ||D x||_1      (Eq. 1)
 * with (D z)_i = z_{i+1} - z_i (reading O2 in DESIGN.md).
 *
 * Functions and the passage each follows:
 *   tvref_prox1d        Eq. 1, solved exactly by the direct
 *                       taut-string method the paper cites (Condat
 *                       2013), restated from SURVEY.md 8(c) item 1.
 *   tvref_prox1d_edges  Eq. 1 with a per-edge weight lam_i (weighted TV,
 *                       north_star only; reading O22): shortest path through
 *                       the tube of half-widths lam_i around the cumulative
 *                       sum of y (taut string), long double.
 *   tvref_codes         segmentation of a solution x: which edges are jumps
 *                       and their signs (support S-bar of D x).
 *   tvref_bwd1d         Eq. 7-8 under reading O12: the Jacobian
 *                       dx/dy is the orthogonal projector onto vectors that
 *                       are constant on the segments of x (segment mean), and
 *                       dx/dlam on segment [a,b) is (s_R - s_L)/(b-a).
 *   tvref_prox2d        Algorithm 1 (Proximal Dykstra), executed
 *                       literally with the O11 index readings.
 *   tvref_bwd2d         reverse mode through the K unrolled iterations of
 *                       Algorithm 1, one adjoint variable per
 *                       variable of the algorithm (Ybar, Pbar, Zbar, Qbar).
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): brute-force sign-pattern
 * enumeration, KKT certificates, closed forms (two-point, unit step,
 * lam_max), the paper's lam=0 identity, SPEC worked examples, dense Eq. 8,
 * central finite differences, 2D separability / global-mean / sum
 * invariants.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ------------------------------------------------------------------------ */
/* 1D prox, scalar lam: direct taut string (SURVEY 8(c).1 restatement).      */
/* vmin/vmax are the lowest/highest admissible values of the current         */
/* segment, umin/umax the corresponding running dual residuals, km/kp the    */
/* last positions where the lower/upper string was pinned.                   */
/* ------------------------------------------------------------------------ */
static void fill_range(double *x, int64_t from, int64_t to_incl, double v)
{
    for (int64_t i = from; i <= to_incl; ++i) x[i] = v;
}

int tvref_prox1d(int64_t n, const double *y, double lam, double *x)
{
    if (n < 1) return 0;
    if (!(lam > 0.0)) {                 /* lam = 0: identity */
        for (int64_t i = 0; i < n; ++i) x[i] = y[i];
        return 0;
    }
    int64_t k = 0, k0 = 0, km = 0, kp = 0;
    double umin = lam, umax = -lam;
    double vmin = y[0] - lam, vmax = y[0] + lam;
    for (;;) {
        while (k == n - 1) {            /* reached the right end */
            if (umin < 0.0) {           /* lower string must drop: emit vmin */
                fill_range(x, k0, km, vmin);
                k0 = km + 1; k = k0; km = k0;
                vmin = y[k]; umin = lam; umax = vmin + umin - vmax;
            } else if (umax > 0.0) {    /* upper string must rise: emit vmax */
                fill_range(x, k0, kp, vmax);
                k0 = kp + 1; k = k0; kp = k0;
                vmax = y[k]; umax = -lam; umin = vmax + umax - vmin;
            } else {                    /* last segment closes at the end */
                vmin += umin / (double)(k - k0 + 1);
                fill_range(x, k0, k, vmin);
                return 0;
            }
        }
        umin += y[k + 1] - vmin;
        if (umin < -lam) {              /* negative jump after km */
            fill_range(x, k0, km, vmin);
            k0 = km + 1; k = k0; kp = k0; km = k0;
            vmin = y[k]; vmax = vmin + 2.0 * lam;
            umin = lam; umax = -lam;
            continue;
        }
        umax += y[k + 1] - vmax;
        if (umax > lam) {               /* positive jump after kp */
            fill_range(x, k0, kp, vmax);
            k0 = kp + 1; k = k0; kp = k0; km = k0;
            vmax = y[k]; vmin = vmax - 2.0 * lam;
            umin = lam; umax = -lam;
            continue;
        }
        k += 1;                         /* no jump yet: extend the segment */
        if (umin >= lam) {
            km = k; vmin += (umin - lam) / (double)(km - k0 + 1); umin = lam;
        }
        if (umax <= -lam) {
            kp = k; vmax += (umax + lam) / (double)(kp - k0 + 1); umax = -lam;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* 1D prox, per-edge lam_i >= 0 (reading O22).  Taut string through the      */
/* tube L_k = S_k - lam_{k-1}, U_k = S_k + lam_{k-1} (k = 1..n-1) from        */
/* (0,0) to (n, S_n), S_k = sum_{j<k} y_j; x_j is the slope on [j, j+1].     */
/* Funnel construction, O(n^2) worst case, long double.                      */
/* ------------------------------------------------------------------------ */
int tvref_prox1d_edges(int64_t n, const double *y, const double *lam, double *x)
{
    if (n < 1) return 0;
    long double *S = (long double *)malloc(sizeof(long double) * (size_t)(n + 1));
    long double *L = (long double *)malloc(sizeof(long double) * (size_t)(n + 1));
    long double *U = (long double *)malloc(sizeof(long double) * (size_t)(n + 1));
    if (!S || !L || !U) { free(S); free(L); free(U); return -1; }
    S[0] = 0.0L;
    for (int64_t k = 1; k <= n; ++k) S[k] = S[k - 1] + (long double)y[k - 1];
    L[0] = U[0] = 0.0L;
    L[n] = U[n] = S[n];
    for (int64_t k = 1; k < n; ++k) {
        L[k] = S[k] - (long double)lam[k - 1];
        U[k] = S[k] + (long double)lam[k - 1];
    }
    int64_t i0 = 0;
    long double X0 = 0.0L;
    while (i0 < n) {
        long double smin = -INFINITY, smax = INFINITY;
        int64_t imin = i0, imax = i0;
        int bent = 0;
        for (int64_t k = i0 + 1; k <= n; ++k) {
            long double lo = (L[k] - X0) / (long double)(k - i0);
            long double hi = (U[k] - X0) / (long double)(k - i0);
            if (lo > smax) {            /* string bends up at upper point imax */
                for (int64_t j = i0; j < imax; ++j) x[j] = (double)smax;
                X0 = U[imax]; i0 = imax; bent = 1; break;
            }
            if (hi < smin) {            /* string bends down at lower point imin */
                for (int64_t j = i0; j < imin; ++j) x[j] = (double)smin;
                X0 = L[imin]; i0 = imin; bent = 1; break;
            }
            if (lo > smin) { smin = lo; imin = k; }
            if (hi < smax) { smax = hi; imax = k; }
        }
        if (!bent) {                    /* straight to the end point */
            long double s = (S[n] - X0) / (long double)(n - i0);
            for (int64_t j = i0; j < n; ++j) x[j] = (double)s;
            i0 = n;
        }
    }
    free(S); free(L); free(U);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Segmentation of a solution: brk[e] = 1 iff edge e (between samples e and  */
/* e+1) separates two segments; sgn[e] = sign(x[e+1] - x[e]).  An edge with  */
/* lam_e = 0 is always a boundary (its dual is pinned to 0; reading O23).     */
/* lam_edges may be NULL (then lam applies to every edge).                   */
/* ------------------------------------------------------------------------ */
void tvref_codes(int64_t n, const double *x, const double *lam_edges, double lam,
                 int8_t *brk, int8_t *sgn)
{
    for (int64_t e = 0; e + 1 < n; ++e) {
        double d = x[e + 1] - x[e];
        double le = lam_edges ? lam_edges[e] : lam;
        sgn[e] = (int8_t)((d > 0.0) - (d < 0.0));
        brk[e] = (int8_t)((d != 0.0) || !(le > 0.0));
    }
}

/* ------------------------------------------------------------------------ */
/* 1D backward (Eq. 7-8 under O12).  Segments are maximal runs joined by     */
/* brk = 0 edges.  gy = segment mean of g.  For the lam-gradient each        */
/* segment [a,b) carries dx_j/dlam = (s_R - s_L)/(b-a), s_L = sgn[a-1]       */
/* (0 at the start), s_R = sgn[b-1] (0 at the end):                          */
/*   glam_total = sum_seg (s_R - s_L) * mean_seg(g)                          */
/*   glam_edges[e] = sgn[e] * (mean_left(g) - mean_right(g)) on boundaries,  */
/*                   0 on fused edges.                                       */
/* Any output pointer may be NULL.                                           */
/* ------------------------------------------------------------------------ */
void tvref_bwd1d(int64_t n, const int8_t *brk, const int8_t *sgn, const double *g,
                 double *gy, double *glam_edges, double *glam_total)
{
    double total = 0.0;
    double prev_mean = 0.0;
    int64_t a = 0;
    if (glam_edges) for (int64_t e = 0; e + 1 < n; ++e) glam_edges[e] = 0.0;
    while (a < n) {
        int64_t b = a + 1;
        while (b < n && !brk[b - 1]) ++b;           /* segment [a, b) */
        double s = 0.0;
        for (int64_t j = a; j < b; ++j) s += g[j];
        double mean = s / (double)(b - a);
        if (gy) for (int64_t j = a; j < b; ++j) gy[j] = mean;
        double sL = (a > 0) ? (double)sgn[a - 1] : 0.0;
        double sR = (b < n) ? (double)sgn[b - 1] : 0.0;
        total += (sR - sL) * mean;
        if (glam_edges && a > 0) glam_edges[a - 1] = sL * (prev_mean - mean);
        prev_mean = mean;
        a = b;
    }
    if (glam_total) *glam_total = total;
}

/* ------------------------------------------------------------------------ */
/* 2D: Algorithm 1, literal, H x W plane (row-major).           */
/*   Y(1) = X, P(1) = Q(1) = 0                                              */
/*   for k = 1..K:                                                          */
/*     Z(k)_row(m)   = Prox1D(Y(k)_row(m) + P(k)_row(m), lam)   all rows    */
/*     P(k+1)        = P(k) + Y(k) - Z(k)                                   */
/*     Y(k+1)_col(n) = Prox1D(Z(k)_col(n) + Q(k)_col(n), lam)   all columns */
/*     Q(k+1)        = Q(k) + Z(k) - Y(k+1)                                 */
/*   return Y(K+1)                                                          */
/* Segmentations of every 1D call are returned (nullable) for the backward: */
/*   rbrk/rsgn: [K][H][W-1]   cbrk/csgn: [K][W][H-1]                        */
/* and (nullable, tvref_prox2d_ex) the jumps out[e+1] - out[e] of every 1D   */
/* call's output, same layout (the parity tests' mask audit, reading O13).   */
/* ------------------------------------------------------------------------ */
int tvref_prox2d_ex(int64_t H, int64_t W, const double *X, double lam, int K,
                    double *Yout, int8_t *rbrk, int8_t *rsgn, int8_t *cbrk, int8_t *csgn,
                    double *rjmp, double *cjmp)
{
    int64_t HW = H * W;
    int64_t mx = H > W ? H : W;
    double *Y = (double *)malloc(sizeof(double) * (size_t)HW);
    double *Z = (double *)malloc(sizeof(double) * (size_t)HW);
    double *P = (double *)calloc((size_t)HW, sizeof(double));
    double *Q = (double *)calloc((size_t)HW, sizeof(double));
    double *in = (double *)malloc(sizeof(double) * (size_t)mx);
    double *out = (double *)malloc(sizeof(double) * (size_t)mx);
    int8_t *tb = (int8_t *)malloc((size_t)mx);
    int8_t *ts = (int8_t *)malloc((size_t)mx);
    if (!Y || !Z || !P || !Q || !in || !out || !tb || !ts) {
        free(Y); free(Z); free(P); free(Q); free(in); free(out); free(tb); free(ts);
        return -1;
    }
    memcpy(Y, X, sizeof(double) * (size_t)HW);
    for (int k = 0; k < K; ++k) {
        /* row pass */
        for (int64_t m = 0; m < H; ++m) {
            for (int64_t j = 0; j < W; ++j) in[j] = Y[m * W + j] + P[m * W + j];
            tvref_prox1d(W, in, lam, out);
            for (int64_t j = 0; j < W; ++j) Z[m * W + j] = out[j];
            tvref_codes(W, out, NULL, lam, tb, ts);
            for (int64_t e = 0; e + 1 < W; ++e) {
                int64_t o = ((int64_t)k * H + m) * (W - 1) + e;
                if (rbrk) rbrk[o] = tb[e];
                if (rsgn) rsgn[o] = ts[e];
                if (rjmp) rjmp[o] = out[e + 1] - out[e];
            }
        }
        for (int64_t i = 0; i < HW; ++i) P[i] = P[i] + Y[i] - Z[i];
        /* column pass */
        for (int64_t c = 0; c < W; ++c) {
            for (int64_t i = 0; i < H; ++i) in[i] = Z[i * W + c] + Q[i * W + c];
            tvref_prox1d(H, in, lam, out);
            for (int64_t i = 0; i < H; ++i) Y[i * W + c] = out[i];
            tvref_codes(H, out, NULL, lam, tb, ts);
            for (int64_t e = 0; e + 1 < H; ++e) {
                int64_t o = ((int64_t)k * W + c) * (H - 1) + e;
                if (cbrk) cbrk[o] = tb[e];
                if (csgn) csgn[o] = ts[e];
                if (cjmp) cjmp[o] = out[e + 1] - out[e];
            }
        }
        for (int64_t i = 0; i < HW; ++i) Q[i] = Q[i] + Z[i] - Y[i];
    }
    memcpy(Yout, Y, sizeof(double) * (size_t)HW);
    free(Y); free(Z); free(P); free(Q); free(in); free(out); free(tb); free(ts);
    return 0;
}

int tvref_prox2d(int64_t H, int64_t W, const double *X, double lam, int K,
                 double *Yout, int8_t *rbrk, int8_t *rsgn, int8_t *cbrk, int8_t *csgn)
{
    return tvref_prox2d_ex(H, W, X, lam, K, Yout, rbrk, rsgn, cbrk, csgn, NULL, NULL);
}

/* ------------------------------------------------------------------------ */
/* 2D backward: reverse mode through the K unrolled iterations,     */
/* statement by statement, with the Jacobian of every 1D call taken from    */
/* the given segmentation (tvref_bwd1d).  Adjoint variables:                */
/*   Yb (of Y(k+1)), Pb (of P(k+1)), Qb (of Q(k+1)), Zb (of Z(k)).          */
/* Start: Yb = G, Pb = Qb = 0 (P(K+1), Q(K+1) are not outputs).             */
/* For k = K..1, reversing                                                   */
/*   (4) Q(k+1) = Q(k) + Z(k) - Y(k+1):  Zb = Qb; Yb -= Qb; (Qb carries)     */
/*   (3) Y(k+1) = prox_cols(Z(k) + Q(k)): Bb = J_col^T Yb; Zb += Bb; Qb += Bb */
/*   (2) P(k+1) = P(k) + Y(k) - Z(k):    Zb -= Pb; Yb(k) = Pb; (Pb carries) */
/*   (1) Z(k) = prox_rows(Y(k) + P(k)):   Ab = J_row^T Zb; Yb += Ab; Pb += Ab */
/* X-bar = Yb after k = 1.  Each prox also adds <its adjoint, dx/dlam>.      */
/* ------------------------------------------------------------------------ */
int tvref_bwd2d(int64_t H, int64_t W, int K,
                const int8_t *rbrk, const int8_t *rsgn,
                const int8_t *cbrk, const int8_t *csgn,
                const double *G, double *GX, double *glam)
{
    int64_t HW = H * W;
    int64_t mx = H > W ? H : W;
    double *Yb = (double *)malloc(sizeof(double) * (size_t)HW);
    double *Pb = (double *)calloc((size_t)HW, sizeof(double));
    double *Qb = (double *)calloc((size_t)HW, sizeof(double));
    double *Zb = (double *)malloc(sizeof(double) * (size_t)HW);
    double *in = (double *)malloc(sizeof(double) * (size_t)mx);
    double *out = (double *)malloc(sizeof(double) * (size_t)mx);
    if (!Yb || !Pb || !Qb || !Zb || !in || !out) {
        free(Yb); free(Pb); free(Qb); free(Zb); free(in); free(out);
        return -1;
    }
    memcpy(Yb, G, sizeof(double) * (size_t)HW);
    double lamb = 0.0;
    for (int k = K - 1; k >= 0; --k) {
        /* (4) */
        for (int64_t i = 0; i < HW; ++i) { Zb[i] = Qb[i]; Yb[i] -= Qb[i]; }
        /* (3) column prox: Bb = J^T Yb, added to Zb and Qb */
        for (int64_t c = 0; c < W; ++c) {
            for (int64_t i = 0; i < H; ++i) in[i] = Yb[i * W + c];
            double lt = 0.0;
            int64_t o = ((int64_t)k * W + c) * (H - 1);
            tvref_bwd1d(H, cbrk + o, csgn + o, in, out, NULL, &lt);
            lamb += lt;
            for (int64_t i = 0; i < H; ++i) {
                Zb[i * W + c] += out[i];
                Qb[i * W + c] += out[i];
            }
        }
        /* (2) */
        for (int64_t i = 0; i < HW; ++i) { Zb[i] -= Pb[i]; Yb[i] = Pb[i]; }
        /* (1) row prox: Ab = J^T Zb, added to Yb (of Y(k)) and Pb (of P(k)) */
        for (int64_t m = 0; m < H; ++m) {
            double lt = 0.0;
            int64_t o = ((int64_t)k * H + m) * (W - 1);
            tvref_bwd1d(W, rbrk + o, rsgn + o, Zb + m * W, out, NULL, &lt);
            lamb += lt;
            for (int64_t j = 0; j < W; ++j) {
                Yb[m * W + j] += out[j];
                Pb[m * W + j] += out[j];
            }
        }
    }
    memcpy(GX, Yb, sizeof(double) * (size_t)HW);
    if (glam) *glam = lamb;
    free(Yb); free(Pb); free(Qb); free(Zb); free(in); free(out);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Batched drivers over independent rows / planes with a plain pthread      */
/* split (the timed CPU baseline, bench.py cpu_baseline).  Row b of a 1D    */
/* batch lives at y + b*n; lam per row (lam_rows) or per edge (lam_edges,   */
/* [batch][n-1]); codes [batch][n-1].  2D plane p at X + p*H*W with lam[p].  */
/* ------------------------------------------------------------------------ */
typedef struct {
    int kind;                  /* 0 = 1D fwd, 1 = 1D bwd, 2 = 2D fwd, 3 = 2D bwd */
    int64_t lo, hi, n, H, W;
    int K;
    const double *in, *lam, *g;
    double *out, *out2;
    double *j1, *j2;
    int8_t *b1, *s1, *b2, *s2;
    const int8_t *cb1, *cs1, *cb2, *cs2;
    int per_edge;
    int status;
} tvref_job_t;

static void *tvref_worker(void *arg)
{
    tvref_job_t *j = (tvref_job_t *)arg;
    for (int64_t r = j->lo; r < j->hi; ++r) {
        if (j->kind == 0) {
            int64_t n = j->n, m = n > 1 ? n - 1 : 0;
            const double *le = j->per_edge ? j->lam + r * m : NULL;
            double l = j->per_edge ? 0.0 : j->lam[r];
            int st = le ? tvref_prox1d_edges(n, j->in + r * n, le, j->out + r * n)
                        : tvref_prox1d(n, j->in + r * n, l, j->out + r * n);
            if (st) j->status = st;
            if (j->b1) tvref_codes(n, j->out + r * n, le, l, j->b1 + r * m, j->s1 + r * m);
        } else if (j->kind == 1) {
            int64_t n = j->n, m = n > 1 ? n - 1 : 0;
            tvref_bwd1d(n, j->cb1 + r * m, j->cs1 + r * m, j->g + r * n,
                        j->out + r * n,
                        j->per_edge ? j->out2 + r * m : NULL,
                        j->per_edge ? NULL : j->out2 + r);
        } else if (j->kind == 2) {
            int64_t HW = j->H * j->W;
            int64_t rs = (int64_t)j->K * j->H * (j->W - 1);
            int64_t cs = (int64_t)j->K * j->W * (j->H - 1);
            int st = tvref_prox2d_ex(j->H, j->W, j->in + r * HW, j->lam[r], j->K, j->out + r * HW,
                                     j->b1 ? j->b1 + r * rs : NULL, j->s1 ? j->s1 + r * rs : NULL,
                                     j->b2 ? j->b2 + r * cs : NULL, j->s2 ? j->s2 + r * cs : NULL,
                                     j->j1 ? j->j1 + r * rs : NULL, j->j2 ? j->j2 + r * cs : NULL);
            if (st) j->status = st;
        } else {
            int64_t HW = j->H * j->W;
            int64_t rs = (int64_t)j->K * j->H * (j->W - 1);
            int64_t cs = (int64_t)j->K * j->W * (j->H - 1);
            int st = tvref_bwd2d(j->H, j->W, j->K, j->cb1 + r * rs, j->cs1 + r * rs,
                                 j->cb2 + r * cs, j->cs2 + r * cs, j->g + r * HW,
                                 j->out + r * HW, j->out2 + r);
            if (st) j->status = st;
        }
    }
    return NULL;
}

static int tvref_run(tvref_job_t proto, int64_t count, int nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > count) nthreads = (int)(count > 0 ? count : 1);
    tvref_job_t jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = proto;
        jobs[t].lo = count * t / nthreads;
        jobs[t].hi = count * (t + 1) / nthreads;
        jobs[t].status = 0;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, tvref_worker, &jobs[t]);
    tvref_worker(&jobs[0]);
    int st = jobs[0].status;
    for (int t = 1; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        if (jobs[t].status) st = jobs[t].status;
    }
    return st;
}

int tvref_prox1d_batch(int64_t batch, int64_t n, const double *y, const double *lam,
                       int per_edge, double *x, int8_t *brk, int8_t *sgn, int nthreads)
{
    tvref_job_t j; memset(&j, 0, sizeof j);
    j.kind = 0; j.n = n; j.in = y; j.lam = lam; j.per_edge = per_edge; j.out = x;
    j.b1 = brk; j.s1 = sgn;
    return tvref_run(j, batch, nthreads);
}

int tvref_bwd1d_batch(int64_t batch, int64_t n, const int8_t *brk, const int8_t *sgn,
                      const double *g, double *gy, double *glam, int per_edge, int nthreads)
{
    tvref_job_t j; memset(&j, 0, sizeof j);
    j.kind = 1; j.n = n; j.cb1 = brk; j.cs1 = sgn; j.g = g; j.out = gy; j.out2 = glam;
    j.per_edge = per_edge;
    return tvref_run(j, batch, nthreads);
}

int tvref_prox2d_batch_ex(int64_t planes, int64_t H, int64_t W, const double *X, const double *lam,
                          int K, double *Y, int8_t *rbrk, int8_t *rsgn, int8_t *cbrk, int8_t *csgn,
                          double *rjmp, double *cjmp, int nthreads)
{
    tvref_job_t j; memset(&j, 0, sizeof j);
    j.kind = 2; j.H = H; j.W = W; j.K = K; j.in = X; j.lam = lam; j.out = Y;
    j.b1 = rbrk; j.s1 = rsgn; j.b2 = cbrk; j.s2 = csgn; j.j1 = rjmp; j.j2 = cjmp;
    return tvref_run(j, planes, nthreads);
}

int tvref_prox2d_batch(int64_t planes, int64_t H, int64_t W, const double *X, const double *lam,
                       int K, double *Y, int8_t *rbrk, int8_t *rsgn, int8_t *cbrk, int8_t *csgn,
                       int nthreads)
{
    return tvref_prox2d_batch_ex(planes, H, W, X, lam, K, Y, rbrk, rsgn, cbrk, csgn, NULL, NULL, nthreads);
}

int tvref_bwd2d_batch(int64_t planes, int64_t H, int64_t W, int K,
                      const int8_t *rbrk, const int8_t *rsgn, const int8_t *cbrk, const int8_t *csgn,
                      const double *G, double *GX, double *glam, int nthreads)
{
    tvref_job_t j; memset(&j, 0, sizeof j);
    j.kind = 3; j.H = H; j.W = W; j.K = K; j.cb1 = rbrk; j.cs1 = rsgn; j.cb2 = cbrk; j.cs2 = csgn;
    j.g = G; j.out = GX; j.out2 = glam;
    return tvref_run(j, planes, nthreads);
}
