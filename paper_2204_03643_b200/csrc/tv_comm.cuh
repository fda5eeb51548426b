// tv_comm.cuh -- line-group communication for the PN solver.
//
// A line is held by LPR lanes of each of WPL warps (NL = LPR*WPL lanes, line lane
// index w*LPR + l).  WPL == 1: the group is LPR consecutive lanes of one warp and
// every operation is a width-LPR warp shuffle / vote.  WPL > 1: the block is
// exactly one line (LPR == 32); warp-level results are combined across the WPL
// warps through a small shared-memory scratch and __syncthreads.  Each call site
// owns a slot S, so a slot is rewritten only after at least one other barrier.
#pragma once
#include "tv_common.cuh"

namespace tvp {

constexpr int kCommSlots = 16;

template <typename T, int LPR, int WPL>
struct Comm {
    static constexpr bool kCluster = false;
    int l;      // lane within the warp group [0, LPR)
    int w;      // warp within the line [0, WPL)
    T* sv;      // [kCommSlots][3][WPL]   (WPL > 1)
    int* si;    // [kCommSlots][WPL]      (WPL > 1)

    __device__ __forceinline__ bool first_lane() const { return (WPL == 1 || w == 0) && l == 0; }
    __device__ __forceinline__ T& V(int s, int j, int ww) const { return sv[(s * 3 + j) * WPL + ww]; }
    __device__ __forceinline__ int& I(int s, int ww) const { return si[s * WPL + ww]; }

    // value held by line lane - 1 (0 at line lane 0)
    template <int S>
    __device__ __forceinline__ T prev(T v) const {
        T p = shup<LPR>(v, 1);
        if (WPL > 1) {
            if (l == LPR - 1) V(S, 0, w) = v;
            __syncthreads();
            if (l == 0 && w > 0) p = V(S, 0, w - 1);
        }
        return first_lane() ? T(0) : p;
    }
    // value held by line lane + 1 (unspecified at the last lane)
    template <int S>
    __device__ __forceinline__ T next(T v) const {
        T nx = shdn<LPR>(v, 1);
        if (WPL > 1) {
            if (l == 0) V(S, 0, w) = v;
            __syncthreads();
            if (l == LPR - 1 && w + 1 < WPL) nx = V(S, 0, w + 1);
        }
        return nx;
    }
    // both neighbours with one barrier
    template <int S>
    __device__ __forceinline__ void prev_next(T vp, T vn, T& p, T& nx) const {
        p = shup<LPR>(vp, 1);
        nx = shdn<LPR>(vn, 1);
        if (WPL > 1) {
            if (l == LPR - 1) V(S, 0, w) = vp;
            if (l == 0) V(S, 1, w) = vn;
            __syncthreads();
            if (l == 0 && w > 0) p = V(S, 0, w - 1);
            if (l == LPR - 1 && w + 1 < WPL) nx = V(S, 1, w + 1);
        }
        if (first_lane()) p = T(0);
    }

    __device__ __forceinline__ bool any(bool p) const {
        if (WPL > 1) return __syncthreads_or(p) != 0;
        return group_any<LPR>(p);
    }
    __device__ __forceinline__ bool all(bool p) const {
        if (WPL > 1) return __syncthreads_and(p) != 0;
        return group_all<LPR>(p);
    }
    // true iff p on any lane of the warp (loop control; line-uniform values only)
    __device__ __forceinline__ bool uany(bool p) const {
        if (WPL > 1) return p;           // block == line: already uniform
        return __any_sync(FULL, p);
    }

    template <int S>
    __device__ __forceinline__ T sum(T v) const {
        v = group_sum<LPR>(v);
        if (WPL > 1) {
            if (l == 0) V(S, 0, w) = v;
            __syncthreads();
            v = T(0);
#pragma unroll
            for (int i = 0; i < WPL; ++i) v += V(S, 0, i);
        }
        return v;
    }
    template <int S>
    __device__ __forceinline__ void sum3(T& a, T& b, T& c) const {
        a = group_sum<LPR>(a);
        b = group_sum<LPR>(b);
        c = group_sum<LPR>(c);
        if (WPL > 1) {
            if (l == 0) { V(S, 0, w) = a; V(S, 1, w) = b; V(S, 2, w) = c; }
            __syncthreads();
            a = b = c = T(0);
#pragma unroll
            for (int i = 0; i < WPL; ++i) { a += V(S, 0, i); b += V(S, 1, i); c += V(S, 2, i); }
        }
    }
    template <int S>
    __device__ __forceinline__ T max_(T v) const {
        v = group_max<LPR>(v);
        if (WPL > 1) {
            if (l == 0) V(S, 0, w) = v;
            __syncthreads();
            v = V(S, 0, 0);
#pragma unroll
            for (int i = 1; i < WPL; ++i) v = max(v, V(S, 0, i));
        }
        return v;
    }

    // ---- Segmented scans.  The flags of one solver step are the same for all its
    // scans (f = "the lane holds a bound edge"), so the lane geometry of the segments
    // is derived once from a ballot (seg_plan) and each scan then only moves data:
    //   h  = highest flagged lane <= this lane in the group (the segment head), D = l - h;
    //   a Hillis-Steele level d adds the partial of lane l - d iff d <= D, which is
    //   exactly when the flag-carrying form (combine(L, R) = R.f ? R : L + R) adds it,
    //   so the sums are bitwise those of that form, with one shuffle per level;
    //   rs = lowest flagged lane strictly above this lane (reverse broadcast source).
    struct Seg {
        int D;          // adds allowed for levels d <= D
        int h;          // segment head lane (absolute), valid if hh
        bool hh;        // a flagged lane at or below this lane (in the group)
        bool hx;        // a flagged lane strictly below this lane
        int rs;         // lowest flagged lane strictly above (absolute), valid if rf
        bool rf;
        int Dr;         // reverse scans: adds allowed for levels d <= Dr (lowest flagged lane
                        // >= this lane, else the group's last lane, minus this lane)
        uint32_t fm;    // ballot of the flags (whole warp)
    };
    __device__ __forceinline__ Seg seg_plan(bool f) const {
        Seg g;
        const uint32_t lane = threadIdx.x & 31u;
        const uint32_t gb = lane & ~uint32_t(LPR - 1);
        const uint32_t fm = __ballot_sync(FULL, f);
        const uint32_t glo = ~((1u << gb) - 1u);                                     // lanes >= gb
        const uint32_t ghi = (LPR == 32 || gb + LPR == 32) ? 0xffffffffu : ((1u << (gb + LPR)) - 1u);
        const uint32_t le = fm & glo & ((2u << lane) - 1u);                          // flagged, <= lane
        const uint32_t gt = fm & ghi & ~((2u << lane) - 1u);                         // flagged, > lane
        g.hh = le != 0u;
        g.h = g.hh ? 31 - __clz(le) : (int)gb;
        g.D = (int)lane - g.h;
        g.hx = (le & ~(1u << lane)) != 0u;
        g.rf = gt != 0u;
        g.rs = g.rf ? __ffs(gt) - 1 : (int)lane;
        const uint32_t ge = fm & ghi & ~((1u << lane) - 1u);                          // flagged, >= lane
        g.Dr = (ge ? __ffs(ge) - 1 : (int)(gb + LPR - 1)) - (int)lane;
        g.fm = fm;
        return g;
    }

    // Segmented exclusive scan of (a, c): a summed; c a sample count with c == E on
    // lanes without a flag (so its scan is position arithmetic: E per lane since the
    // head plus the head's own count).
    template <int S, int E>
    __device__ __forceinline__ void scan_fwd(const Seg& g, T& a, int& c) const {
        const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
        for (int d = 1; d < LPR; d <<= 1) {
            const T a2 = shup<LPR>(a, d);
            if (d <= g.D) a += a2;
        }
        const int ch = __shfl_sync(FULL, c, g.h);
        const int ci = g.hh ? g.D * E + ch : (g.D + 1) * E;                  // inclusive count
        T ea = shup<LPR>(a, 1);
        int ecf = shup<LPR>(ci | (g.hh ? (1 << 30) : 0), 1);
        if (l == 0) { ea = T(0); ecf = 0; }
        (void)lane;
        if (WPL > 1) {
            if (l == LPR - 1) { V(S, 0, w) = a; I(S, w) = ci | (g.hh ? (1 << 30) : 0); }
            __syncthreads();
            T ca = T(0);
            int cc = 0;
            if constexpr (WPL > 2) {
                // log-depth segmented scan of the WPL warp aggregates on lanes 0..WPL-1
                T xa = (l < WPL) ? V(S, 0, l) : T(0);
                int xc = (l < WPL) ? I(S, l) : 0;
#pragma unroll
                for (int d = 1; d < WPL; d <<= 1) {
                    const T a2 = shup<32>(xa, d);
                    const int c2 = shup<32>(xc, d);
                    if (l >= d && !(xc >> 30)) { xa += a2; xc = (xc & 0x3fffffff) + (c2 & 0x3fffffff) | (c2 & (1 << 30)); }
                }
                ca = __shfl_sync(FULL, xa, w > 0 ? w - 1 : 0);
                cc = __shfl_sync(FULL, xc, w > 0 ? w - 1 : 0) & 0x3fffffff;
                if (w == 0) { ca = T(0); cc = 0; }
            } else {
#pragma unroll
                for (int i = 0; i < WPL - 1; ++i) {
                    if (i < w) {
                        const T ra = V(S, 0, i);
                        const int rcf = I(S, i);
                        if (rcf >> 30) { ca = ra; cc = rcf & 0x3fffffff; } else { ca += ra; cc += rcf & 0x3fffffff; }
                    }
                }
            }
            if (!(ecf >> 30)) { ea += ca; ecf += cc; }
        }
        a = ea;
        c = ecf & 0x3fffffff;
    }
    // Two-warp lines: scan_fwd, the first-segment values and scan_rev_c in ONE block exchange.
    // The forward carry only reaches warp 1 and the reverse carry only warp 0, so each warp
    // publishes its forward tail aggregate and the record of its first flagged lane (in-warp
    // forward prefix, head numerator, bit index, lambda / |y| bounds, flagless head sums);
    // warp 0 recomputes warp 1's first-segment value with exactly warp 1's operations (so
    // the shared segment's value is bitwise one value).  In: this lane's P1 tail sum s and
    // count ctail, head numerator numf, first bound index fb, lmaxl, yabs.  Out: fv, the
    // reverse carry (vh, ah) and cur as scan_rev_c.
    template <int S, int E>
    __device__ __forceinline__ void scan_all2(const Seg& g, bool fl, T s, int ctail, T numf, int fb, T lmaxl,
                                              T yabs, T& fv, T& vh, T& ah, T& cur) const {
        static_assert(WPL == 2, "two-warp lines");
        constexpr int M = 0x3fffffff, F = 1 << 30;
        const int lane = (int)(threadIdx.x & 31u);
        // forward in-warp part (scan_fwd)
        T a = s;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shup<32>(a, d);
            if (d <= g.D) a += a2;
        }
        const int ch = __shfl_sync(FULL, ctail, g.h);
        const int ci = g.hh ? g.D * E + ch : (g.D + 1) * E;
        T ea = shup<32>(a, 1);
        int ecf = shup<32>(ci | (g.hh ? F : 0), 1);
        if (l == 0) { ea = T(0); ecf = 0; }
        // reverse in-warp sums of the flagless lanes' (s, |y|)
        T ra = fl ? T(0) : s, rb = fl ? T(0) : yabs;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shdn<32>(ra, d), b2 = shdn<32>(rb, d);
            if (d <= g.Dr) { ra += a2; rb += b2; }
        }
        T era = shdn<32>(ra, 1), erb = shdn<32>(rb, 1);
        if (l == 31) { era = T(0); erb = T(0); }
        // the warp's first flagged lane
        const int ff = g.fm ? __ffs(g.fm) - 1 : 32;
        const int src = g.fm ? ff : 0;
        const T ea_f = __shfl_sync(FULL, ea, src), nu_f = __shfl_sync(FULL, numf, src);
        const T lm_f = __shfl_sync(FULL, lmaxl, src), ya_f = __shfl_sync(FULL, yabs, src);
        const int ecf_f = __shfl_sync(FULL, ecf, src), fb_f = __shfl_sync(FULL, fb, src);
        if (l == 31) { V(S, 0, w) = a; I(S, w) = ci | (g.hh ? F : 0); }
        if (l == 0) {
            V(S, 1, w) = ea_f; V(S, 2, w) = nu_f;
            V(S + 1, 0, w) = lm_f; V(S + 1, 1, w) = ya_f; V(S + 1, 2, w) = ra;
            V(S + 2, 0, w) = rb;
            I(S + 1, w) = ecf_f;
            I(S + 2, w) = ff | (fb_f << 8);
        }
        __syncthreads();
        const T ra0 = V(S, 0, 0);                     // warp 0's forward tail aggregate
        const int rc0 = I(S, 0);
        if (w == 1 && !(ecf >> 30)) { ea += ra0; ecf += rc0 & M; }
        fv = (numf + ea) * rcp_(T(fb + 1 + (ecf & M)));
        // reverse carry
        const T vhl = fl ? (numf - T(fb + 1) * fv) : T(0);
        const T ahl = fl ? (lmaxl + T(fb + 1) * fabs(fv)) + yabs : T(0);
        T c = __shfl_sync(FULL, fv, g.rs), v = __shfl_sync(FULL, vhl, g.rs), h = __shfl_sync(FULL, ahl, g.rs);
        int nn = g.rs - lane - 1;
        if (!g.rf) {
            if (w == 0) {
                T cs1 = V(S, 1, 1);
                int cc1 = I(S + 1, 1);
                if (!(cc1 >> 30)) { cs1 += ra0; cc1 += rc0 & M; }
                const int pk = I(S + 2, 1), ff1 = pk & 255, fb1 = pk >> 8;
                const T nu1 = V(S, 2, 1);
                const T fv1 = (nu1 + cs1) * rcp_(T(fb1 + 1 + (cc1 & M)));
                c = fv1;
                v = nu1 - T(fb1 + 1) * fv1;
                h = (V(S + 1, 0, 1) + T(fb1 + 1) * fabs(fv1)) + V(S + 1, 1, 1);
                era += V(S + 1, 2, 1);
                erb += V(S + 2, 0, 1);
                nn = 31 - lane + ff1;
            } else {                                   // past the line's last flagged lane
                c = T(0); v = T(0); h = T(0); nn = 0;
            }
        }
        cur = c;
        vh = v + era - T(E) * T(nn) * c;
        ah = h + erb + T(E) * T(nn) * fabs(c);
    }

    // Reverse segmented exclusive scan of two summed values (a, b): each line lane gets the
    // sums over the lanes strictly to its right up to and including the nearest flagged one
    // (up to the line's end if none) -- the mirror image of a forward segmented scan.
    template <int S>
    __device__ __forceinline__ void scan_rev2(const Seg& g, T& a, T& b) const {
#pragma unroll
        for (int d = 1; d < LPR; d <<= 1) {
            const T a2 = shdn<LPR>(a, d), b2 = shdn<LPR>(b, d);
            if (d <= g.Dr) { a += a2; b += b2; }
        }
        T ea = shdn<LPR>(a, 1), eb = shdn<LPR>(b, 1);
        if (l == LPR - 1) { ea = T(0); eb = T(0); }
        if (WPL > 1) {
            if (l == 0) { V(S, 0, w) = a; V(S, 1, w) = b; I(S, w) = (int)(g.fm != 0u); }
            __syncthreads();
            T ca = T(0), cb = T(0);
            if constexpr (WPL > 2) {
                T xa = (l < WPL) ? V(S, 0, l) : T(0), xb = (l < WPL) ? V(S, 1, l) : T(0);
                int xf = (l < WPL) ? I(S, l) : 0;
#pragma unroll
                for (int d = 1; d < WPL; d <<= 1) {
                    const T a2 = shdn<32>(xa, d), b2 = shdn<32>(xb, d);
                    const int f2 = shdn<32>(xf, d);
                    if (l + d < WPL && !xf) { xa += a2; xb += b2; xf = f2; }
                }
                ca = __shfl_sync(FULL, xa, w + 1 < WPL ? w + 1 : 0);
                cb = __shfl_sync(FULL, xb, w + 1 < WPL ? w + 1 : 0);
                if (w + 1 >= WPL) { ca = T(0); cb = T(0); }
            } else {
#pragma unroll
                for (int i = WPL - 1; i >= 1; --i) {
                    if (i > w) {
                        if (I(S, i)) { ca = V(S, 0, i); cb = V(S, 1, i); } else { ca += V(S, 0, i); cb += V(S, 1, i); }
                    }
                }
            }
            if (!g.rf) { ea += ca; eb += cb; }
        }
        a = ea;
        b = eb;
    }
    // Value of the nearest flagged line lane strictly to the right (0 if none): one
    // shuffle from the plan's source lane.
    template <int S>
    __device__ __forceinline__ T scan_rev(const Seg& g, T v) const {
        T e = __shfl_sync(FULL, v, g.rs);
        if (!g.rf) e = T(0);
        if (WPL > 1) {
            // the warp's inclusive-from-the-left value: its lowest flagged lane's v
            const T vf = __shfl_sync(FULL, v, g.fm ? __ffs(g.fm) - 1 : 0);
            if (l == 0) { V(S, 0, w) = vf; I(S, w) = g.fm != 0u; }
            __syncthreads();
            if constexpr (WPL > 2) {
                // nearest flagged warp strictly to the right: log-depth on lanes 0..WPL-1
                T xv = (l < WPL) ? V(S, 0, l) : T(0);
                int xf = (l < WPL) ? I(S, l) : 0;
                if (!xf) xv = T(0);
#pragma unroll
                for (int d = 1; d < WPL; d <<= 1) {
                    const T v2 = shdn<32>(xv, d);
                    const int f2 = shdn<32>(xf, d);
                    if (l + d < WPL && !xf) { xv = v2; xf = f2; }
                }
                const T r = __shfl_sync(FULL, xv, w + 1 < WPL ? w + 1 : 0);
                if (!g.rf && w + 1 < WPL) e = r;
            } else if (!g.rf) {
                // nearest flagged warp to the right: the last assignment (lowest i > w) wins
#pragma unroll
                for (int i = WPL - 1; i >= 1; --i) {
                    if (i > w && I(S, i)) e = V(S, 0, i);
                }
            }
        }
        return e;
    }
};

}  // namespace tvp
