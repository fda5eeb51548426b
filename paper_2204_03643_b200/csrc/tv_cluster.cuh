// tv_cluster.cuh -- f2 for planes too large for one CTA (65..224 samples per side, fp32):
// the fused 2D Dykstra forward (Alg. 1) and its reverse mode on a
// thread-block cluster of NC CTAs whose shared memories hold the whole plane state
// across all K iterations (C5's 224^2 planes).
//
// Partition.  CTA j of the cluster owns rows [j*RB, j*RB + RB) and columns
// [j*CB, j*CB + CB) of the plane (RB, CB = ceil(H/NC), ceil(W/NC) rounded up to 4).
// In the forward, P is only used by row passes and Q only by column passes (Alg. 1
// lines 3-10), so each lives with its owner, and every CTA stores its own LINES
// contiguously: rows Yr, Pr [RB][PR], columns Zc, Qc [CB][PH] (column-major), so a line
// is read and written the same way in both orientations (8-byte accesses; lane l's E
// contiguous samples; conflict-free).  Only the Y / Z plane changes hands:
//   row pass k    Yr, Pr -> Z in place in Yr, P <- A - Z;  CTA barrier;  exchange:
//                 every 4 x 1 block Yr[4b..4b+3][c] goes as ONE 16-byte st.shared::cluster
//                 to Zc_d[c - d*CB][r0 + 4b ..] of the column owner d;  cluster barrier;
//   column pass k Zc, Qc -> Y in place in Zc, Q <- B - Y;  CTA barrier;  the transposed
//                 exchange back into the owners' Yr (or Y to HBM after pass K);
//                 cluster barrier.
// HBM sees X once, Y once and the saved masks: 10 B/px instead of ~120 B/px staged.
// The reverse mode is the same exchange with the two adjoint planes A (= Ybar = Pbar)
// and B (= Zbar = Qbar): the column adjoint reads Ac, Bc and writes Bc, which goes to
// the owners' Br; the row adjoint reads Br, Ar and writes Ar, which goes to the owners' Ac.
//
// Every line is solved by the same solve_line / seg_mean as the staged passes, with the
// same lane geometry (LPR = 16 lanes x E samples; two lines per warp) and the same operand
// order (A = Y + P, P = A - Z, ...), so outputs, saved masks and gradients are bitwise
// those of the staged path (tests/test_gpu_parity_2d.py).  Forward lines are handed out
// to warps dynamically (a shared counter per pass): PN iteration counts vary per line and
// each pass ends at a cluster barrier.
#pragma once
#include "tv_kernels.cuh"
#include "tv_cl_util.cuh"

namespace tvp {

// Geometry of one CTA's share of a plane (host and device).
struct ClGeo {
    int RB, CB, PR, PH, NLM;
};
__host__ __device__ inline ClGeo cl_geo(int H, int W, int NC) {
    ClGeo g;
    g.RB = (((H + NC - 1) / NC) + 3) & ~3;
    g.CB = (((W + NC - 1) / NC) + 3) & ~3;
    g.PR = (W + 3) & ~3;
    g.PH = (H + 3) & ~3;
    g.NLM = g.RB > g.CB ? g.RB : g.CB;
    return g;
}
// Dynamic shared memory: two row planes [RB][PR], two column planes [CB][PH], and in the
// forward the warm-start bits [2 orientations][NLM lines][16 lanes x (up, down)] and a
// 32-word mask buffer per warp.
template <typename T>
__host__ __device__ inline size_t cl_smem_bytes(int H, int W, int NC, int WPB, bool fwd) {
    const ClGeo g = cl_geo(H, W, NC);
    size_t b = (size_t)2 * g.RB * g.PR * sizeof(T) + (size_t)2 * g.CB * g.PH * sizeof(T);
    if (fwd) b += (size_t)2 * g.NLM * 32 * 4 + (size_t)WPB * 32 * 4;
    return b;
}

// Lane l's E contiguous samples of a line (8-byte shared-memory accesses; samples past
// n read as 0, as in the staged passes).
template <int E>
__device__ __forceinline__ void line_ld(const float* line, int l, int n, bool valid, float (&v)[E]) {
    static_assert(E % 2 == 0, "pairs");
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
        const int i = l * E + 2 * j;
        float2 f = make_float2(0.f, 0.f);
        if (valid && i < n) f = *reinterpret_cast<const float2*>(line + i);
        v[2 * j] = f.x;
        v[2 * j + 1] = (i + 1 < n) ? f.y : 0.f;
    }
}
template <int E>
__device__ __forceinline__ void line_st(float* line, int l, int n, const float (&v)[E]) {
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
        const int i = l * E + 2 * j;
        if (i + 1 < n) *reinterpret_cast<float2*>(line + i) = make_float2(v[2 * j], v[2 * j + 1]);
        else if (i < n) line[i] = v[2 * j];
    }
}

// Transposing exchange of the lines a CTA owns into their owners in the other
// orientation.  src: my nsrc lines [nsrc][ps] of length len (the other orientation's
// index); block (b, x) = src[4b .. 4b+3][x] goes to line (x - d*DB) of CTA d = x / DB at
// offset off0 + 4b, one 16-byte remote store; dst_s = the destination buffer's shared
// address (same in every CTA), pd its pitch.  dst_g (nullable): write to HBM instead,
// rows x of a plane of width gw, columns off0 + 4b.. (the final Y / grad_X).
__device__ __forceinline__ void cl_exchange(const float* src, int nsrc, int ps, int len, int DB, uint32_t dst_s,
                                            int pd, int off0, float* dst_g, int gw, int nth) {
    const int nb = (nsrc + 3) >> 2;
    for (int it = threadIdx.x; it < nb * len; it += nth) {
        const int b = it / len, x = it - b * len;
        const float* s = src + 4 * b * ps + x;
        const float v0 = s[0], v1 = s[ps], v2 = s[2 * ps], v3 = s[3 * ps];
        if (dst_g) {
            float* g = dst_g + (int64_t)x * gw + off0 + 4 * b;
            const int m = nsrc - 4 * b;
            if (m >= 4 && ((reinterpret_cast<uintptr_t>(g) & 15) == 0)) {
                *reinterpret_cast<float4*>(g) = make_float4(v0, v1, v2, v3);
                continue;
            }
            g[0] = v0;
            if (m > 1) g[1] = v1;
            if (m > 2) g[2] = v2;
            if (m > 3) g[3] = v3;
        } else {
            const int d = x / DB;
            const uint32_t ra = cl_map(dst_s + (uint32_t)(((x - d * DB) * pd + off0 + 4 * b) * 4), d);
            cl_st4(ra, v0, v1, v2, v3);
        }
    }
}

// Push a solved line PAIR to the owners of the other orientation, straight from
// registers: lanes l and l + 16 hold samples x = l*E + q of lines 2t and 2t + 1; after one
// shuffle per pair of samples each lane owns E/2 sample pairs (x, line 2t / 2t + 1) and
// stores each as one 8-byte st.shared::cluster to line (x - d*DB) of CTA d = x / DB at
// offset off (= the pair's first line in that CTA's line coordinates).  Stores overlap
// the other warps' solves; the pass ends at a cluster barrier.
template <int E>
__device__ __forceinline__ void pair_push(const float (&w)[E], int l, int grp, int n, int DB, uint32_t dst_s, int pd,
                                          int off) {
    constexpr int HE = E / 2;
    const int x0 = l * E + (grp ? HE : 0);
    int d = x0 / DB;
    int xr = x0 - d * DB;
#pragma unroll
    for (int j = 0; j < HE; ++j) {
        const float send = grp ? w[j] : w[HE + j];
        const float recv = __shfl_xor_sync(FULL, send, 16);
        const float a = grp ? recv : w[j];
        const float b = grp ? w[HE + j] : recv;
        if (j > 0 && xr >= DB) { xr -= DB; ++d; }
        if (x0 + j < n) cl_st2(cl_map(dst_s + (uint32_t)((xr * pd + off) * 4), d), a, b);
        ++xr;
    }
}

template <typename T, int E, int NC, int WPB, bool LSP>
__global__ void __launch_bounds__(WPB * 32, 512 / (WPB * 32)) k_plane_fwd_cl(PlaneFwdArgs<T> a) {
    static_assert(sizeof(T) == 4, "fp32 planes");
    constexpr int LPR = 16, G = 2;
    extern __shared__ __align__(16) unsigned char smraw_[];
    __shared__ int s_next[2];                        // dynamic line-pair counters (per orientation)
    const int H = a.H, W = a.W, K = a.K;
    const ClGeo g = cl_geo(H, W, NC);
    const int RB = g.RB, CB = g.CB, PR = g.PR, PH = g.PH;
    float* Yr = reinterpret_cast<float*>(smraw_);
    float* Pr = Yr + RB * PR;
    float* Zc = Pr + RB * PR;
    float* Qc = Zc + CB * PH;
    uint32_t* wbits = reinterpret_cast<uint32_t*>(Qc + CB * PH);     // [2][NLM][32]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    uint32_t* mwb = wbits + 2 * g.NLM * 32 + warp * 32;
    const int nth = WPB * 32;
    const int rank = (int)cl_rank();
    const int r0 = rank * RB, nr = max(0, min(RB, H - r0));          // my rows
    const int c0 = rank * CB, ncl = max(0, min(CB, W - c0));         // my columns
    const int64_t HW = (int64_t)H * W;
    const int64_t rset = a.planes * H * a.mwr, cset = a.planes * W * a.mwc;
    const uint32_t zc_s = smem_u32(Zc), yr_s = smem_u32(Yr);
    const Comm<float, LPR, 1> Cm{l, 0, nullptr, nullptr};
    if (threadIdx.x == 0) s_next[0] = s_next[1] = 0;
    // padding samples (past the line ends) are read but never used: define them
    for (int i = threadIdx.x; i < 2 * RB * PR + 2 * CB * PH; i += nth) Yr[i] = 0.f;
    cl_sync();                                       // every CTA of the cluster is running
    for (int64_t p = cl_id(); p < a.planes; p += cl_num()) {
        const float lamp = line_lambda(a.lam, a.lam_mode, a.lam_scalar, p, 1, a.C);
        const bool lz = !(lamp > 0.f);
        // Y^(1) = X: my rows
        const float* Xp = a.X + p * HW + (int64_t)r0 * W;
        if ((W & 3) == 0 && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0)) {
            const int w4 = W >> 2;
            for (int i = threadIdx.x; i < nr * w4; i += nth) {
                const int r = i / w4, c = (i - r * w4) * 4;
                const float4 v = __ldg(reinterpret_cast<const float4*>(Xp) + i);
                *reinterpret_cast<float4*>(Yr + r * PR + c) = v;
            }
        } else {
            for (int i = threadIdx.x; i < nr * W; i += nth) {
                const int r = i / W, c = i - r * W;
                Yr[r * PR + c] = __ldg(Xp + i);
            }
        }
        __syncthreads();
        for (int k = 1; k <= K; ++k) {
#pragma unroll 1
            for (int o = 0; o < 2; ++o) {            // 0: row pass (lines 3-6), 1: column pass (lines 7-10)
                const int n = o ? H : W;
                const int nl = o ? ncl : nr;
                float* yb = o ? Zc : Yr;
                float* cb = o ? Qc : Pr;
                const int pitch = o ? PH : PR;
                uint32_t* wb = wbits + o * g.NLM * 32;
                const bool cold = k == 1;
                const bool last = o == 1 && k == K;      // Y^(K+1) goes to HBM; Q^(K) is never read
                const int pass = 2 * (k - 1) + o;
                if (threadIdx.x == 0) s_next[1 - o] = 0;     // the other orientation's counter (barrier-separated)
                const int npair = (nl + G - 1) / G;
#pragma unroll 1
                for (;;) {
                    int t = 0;
                    if (lane == 0) t = atomicAdd(&s_next[o], 1);
                    t = __shfl_sync(FULL, t, 0);
                    if (t >= npair) break;
                    const int li = t * G + grp;
                    const bool valid = li < nl;
                    float* ln = yb + (valid ? li : 0) * pitch;
                    float* lc = cb + (valid ? li : 0) * pitch;
                    float y[E], w[E], av[E];
                    line_ld<E>(ln, l, n, valid, av);
                    if (!cold) {
                        float cv[E];
                        line_ld<E>(lc, l, n, valid, cv);
#pragma unroll
                        for (int q = 0; q < E; ++q) av[q] = av[q] + cv[q];
                    } else {
#pragma unroll
                        for (int q = 0; q < E; ++q) av[q] = av[q] + 0.f;   // staged: A = Y + 0 at k = 1
                    }
#pragma unroll
                    for (int q = 0; q < E; ++q) y[q] = av[q];
                    const uint32_t wp0 = (!cold && valid) ? wb[li * 32 + l] : 0u;
                    const uint32_t wn0 = (!cold && valid) ? wb[li * 32 + 16 + l] : 0u;
                    Lam<float, E, false> lm;
                    lm.r = lamp;
                    const int st = solve_line<float, E, LPR, 1, false, LSP>(y, w, lm, n, valid, wp0, wn0, Cm,
                                                                            cold && a.coarse != 0, nullptr, a.ls_after);
                    // codes of the lane's edges: next pass's warm bits and the saved mask
                    const float wnx = shdn<LPR>(w[0], 1);
                    uint32_t up, dn;
                    const int e0 = l * E, wlo = e0 >> 4;
                    const uint32_t code = lane_codes<float, E>(w, wnx, e0, n - 1, lz, up, dn);
                    const int sh = 2 * (e0 & 15);
                    const uint32_t clo = code << sh, chi = sh ? (code >> (32 - sh)) : 0u;
                    if (valid) {
                        wb[li * 32 + l] = up;
                        wb[li * 32 + 16 + l] = dn;
                        if (!last) {
                            float cv[E];
#pragma unroll
                            for (int q = 0; q < E; ++q) cv[q] = av[q] - w[q];
                            line_st<E>(lc, l, n, cv);
                        } else {
                            line_st<E>(ln, l, n, w);     // staged for the coalesced HBM write below
                        }
                        if (l == 0) {
                            if (a.iters_max) atomicMax(a.iters_max + pass, st >= 0 ? (st & 0xffff) : (1 << 20));
                            line_diag(st, a.diag, a.hist ? a.hist + pass * kHistBins : nullptr);
                        }
                    }
                    if (!last) {
                        // Z to the column owners' Zc (rows r0 + 2t, +1) / Y to the row owners' Yr
                        if (o == 0) pair_push<E>(w, l, grp, n, CB, zc_s, PH, r0 + t * G);
                        else pair_push<E>(w, l, grp, n, RB, yr_s, PR, c0 + t * G);
                    }
                    if (a.saved) {
                        const int mw = o ? a.mwc : a.mwr;
                        uint32_t* gw = mwb + grp * 16;
                        gw[l] = 0u;
                        __syncwarp();
                        if (clo) atomicOr(&gw[wlo], clo);
                        if (chi) atomicOr(&gw[wlo + 1], chi);
                        __syncwarp();
                        if (valid && l < mw) {
                            const int64_t off = o ? (int64_t)K * rset + (int64_t)(k - 1) * cset + (p * W + c0 + li) * mw
                                                  : (int64_t)(k - 1) * rset + (p * H + r0 + li) * mw;
                            a.saved[off + l] = gw[l];
                        }
                    }
                    __syncwarp();
                }
                if (last) {
                    __syncthreads();
                    cl_exchange(Zc, ncl, PH, H, RB, 0u, PR, c0, a.Y + p * HW, W, nth);
                }
                cl_sync();                           // every pushed line has landed
            }
        }
    }
}

// Reverse mode through the K passes (a-14) on a cluster: init A = G, B = 0; for
// k = K..1: column adjoint B <- B + colsegmean_k(A - B), row adjoint
// A <- Pbar + rowsegmean_k(B - Pbar) with Pbar = A (0 at k = K); grad_X = A.  The work
// per line is uniform, so lines are assigned statically, and the mask words of a pass
// are loaded into registers before the barrier that precedes it.
template <typename T, int E, int NC, int WPB>
__global__ void __launch_bounds__(WPB * 32, 512 / (WPB * 32)) k_plane_bwd_cl(PlaneBwdArgs<T> a) {
    static_assert(sizeof(T) == 4, "fp32 planes");
    constexpr int LPR = 16, G = 2, MAXR = 2;        // line pairs per warp whose masks are prefetched
    extern __shared__ __align__(16) unsigned char smraw_[];
    const int H = a.H, W = a.W, K = a.K;
    const ClGeo g = cl_geo(H, W, NC);
    const int RB = g.RB, CB = g.CB, PR = g.PR, PH = g.PH;
    float* Ar = reinterpret_cast<float*>(smraw_);
    float* Br = Ar + RB * PR;
    float* Ac = Br + RB * PR;
    float* Bc = Ac + CB * PH;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = lane / LPR, l = lane % LPR;
    const int nth = WPB * 32;
    const int rank = (int)cl_rank();
    const int r0 = rank * RB, nr = max(0, min(RB, H - r0));
    const int c0 = rank * CB, ncl = max(0, min(CB, W - c0));
    const int64_t HW = (int64_t)H * W;
    const int64_t rset = a.planes * H * a.mwr, cset = a.planes * W * a.mwc;
    const int64_t HW2 = H + W;
    const uint32_t ac_s = smem_u32(Ac), br_s = smem_u32(Br);
    // padding samples (past the line ends) are read but never used: define them
    for (int i = threadIdx.x; i < 2 * RB * PR + 2 * CB * PH; i += nth) Ar[i] = 0.f;
    // mask words of the warp's lines of pass (k, o), loaded ahead of the pass
    auto mask_base = [&](int64_t p, int k, int o) -> const uint32_t* {
        return o ? a.saved + (int64_t)K * rset + (int64_t)(k - 1) * cset + (p * W + c0) * a.mwc
                 : a.saved + (int64_t)(k - 1) * rset + (p * H + r0) * a.mwr;
    };
    MaskWin<E> mk[MAXR];
    auto prefetch = [&](int64_t p, int k, int o) {
        const int nl = o ? ncl : nr, mw = o ? a.mwc : a.mwr;
        const uint32_t* mb = mask_base(p, k, o);
#pragma unroll
        for (int rr = 0; rr < MAXR; ++rr) {
            const int li = (warp + rr * WPB) * G + grp;
            if (li < nl && mw > 0) mask_words_ld<E>(mb + li * mw, mw, l * E, mk[rr]);
            else {
#pragma unroll
                for (int j = 0; j <= MaskWin<E>::NS; ++j) mk[rr].w[j] = 0u;
            }
        }
    };
    if (cl_id() < a.planes) prefetch(cl_id(), K, 1);
    cl_sync();
    for (int64_t p = cl_id(); p < a.planes; p += cl_num()) {
        // A = G: my rows -> Ar, and (transposed, 16-byte DSMEM stores) to the column owners' Ac
        const float* Gp = a.G + p * HW;
        for (int i = threadIdx.x; i < nr * W; i += nth) {
            const int r = i / W, c = i - r * W;
            Ar[r * PR + c] = __ldg(Gp + (int64_t)(r0 + r) * W + c);
        }
        __syncthreads();
        cl_exchange(Ar, nr, PR, W, CB, ac_s, PH, r0, nullptr, 0, nth);
        cl_sync();
        for (int k = K; k >= 1; --k) {
#pragma unroll 1
            for (int o = 1; o >= 0; --o) {           // 1: column adjoint, 0: row adjoint
                const int n = o ? H : W;
                const int nl = o ? ncl : nr;
                const float* x1 = o ? Ac : Br;       // v = x1 - x2; x2 <- x2 + segmean(v)
                float* x2 = o ? Bc : Ar;
                const int pitch = o ? PH : PR;
                const bool zero2 = k == K;           // B = 0 (column), Pbar = 0 (row) at k = K
                const int mw = o ? a.mwc : a.mwr;
                const uint32_t* mb = mask_base(p, k, o);
#pragma unroll 1
                for (int t = warp, rr = 0; t * G < nl; t += WPB, ++rr) {
                    const int li = t * G + grp;
                    const bool valid = li < nl;
                    const float* l1 = x1 + (valid ? li : 0) * pitch;
                    float* l2 = x2 + (valid ? li : 0) * pitch;
                    float v[E], bv[E];
                    line_ld<E>(l1, l, n, valid, v);
                    if (!zero2) line_ld<E>(l2, l, n, valid, bv);
                    else {
#pragma unroll
                        for (int q = 0; q < E; ++q) bv[q] = 0.f;
                    }
#pragma unroll
                    for (int q = 0; q < E; ++q) v[q] = v[q] - bv[q];
                    MaskWin<E> m;
                    if (rr < MAXR) {
#pragma unroll
                        for (int j = 0; j <= MaskWin<E>::NS; ++j) m.w[j] = rr == 0 ? mk[0].w[j] : mk[MAXR - 1].w[j];
                    } else if (valid && mw > 0) {
                        mask_words_ld<E>(mb + li * mw, mw, l * E, m);
                    } else {
#pragma unroll
                        for (int j = 0; j <= MaskWin<E>::NS; ++j) m.w[j] = 0u;
                    }
                    uint32_t bnd = 0, pos = 0, neg = 0;
                    if (mw > 0) mask_decode<E>(m, l * E, bnd, pos, neg);
                    bnd |= pin_tail<E>(n - 1 - l * E);
                    float lp = 0.f;
                    seg_mean<float, E, LPR>(v, bnd, pos, neg, l, lp);
                    lp = group_sum<LPR>(lp);
#pragma unroll
                    for (int q = 0; q < E; ++q) v[q] = bv[q] + v[q];
                    if (valid) {
                        if (l == 0 && a.lampart)
                            a.lampart[p * K * HW2 + (k - 1) * HW2 + (o ? H + c0 : r0) + li] = lp;
                        if (o == 0 && k == 1) {
                            float* gx = a.GX + p * HW + (int64_t)(r0 + li) * W;
#pragma unroll
                            for (int q = 0; q < E; ++q)
                                if (l * E + q < n) gx[l * E + q] = v[q];
                        } else {
                            line_st<E>(l2, l, n, v);
                        }
                    }
                    // B to the row owners' Br (columns c0 + 2t, +1) / A to the column owners' Ac
                    if (o == 1) pair_push<E>(v, l, grp, n, RB, br_s, PR, c0 + t * G);
                    else if (k > 1) pair_push<E>(v, l, grp, n, CB, ac_s, PH, r0 + t * G);
                }
                // the next pass's mask words, in flight across the barrier
                if (o == 1) prefetch(p, k, 0);
                else if (k > 1) prefetch(p, k - 1, 1);
                else if (p + cl_num() < a.planes) prefetch(p + cl_num(), K, 1);
                cl_sync();
            }
        }
    }
}

}  // namespace tvp
