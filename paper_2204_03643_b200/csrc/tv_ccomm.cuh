// tv_ccomm.cuh -- line-group communication for a line held by a whole thread-block
// cluster (f4: 1D rows longer than one CTA's registers hold).
//
// CComm<T, WPL, NCTA> has the interface of Comm<T, 32, WPL> (tv_comm.cuh), so the same
// projected-Newton solver (pn_solve / solve_line) and segment-mean backward (seg_mean_c)
// run on it unchanged.  The line is held by NW = NCTA * WPL warps (line lane index
// (rank * WPL + warp) * 32 + lane, E contiguous samples per lane).  Every cross-warp
// operation is: warp-level part with shuffles / votes; the warp's aggregate is stored
// into slot (S, warp) of EVERY CTA of the cluster (lanes d < NCTA each store to CTA d,
// st.shared::cluster); one cluster barrier (release / acquire); each warp then combines
// the NW aggregates from its own shared memory -- lanes hold Q = ceil(NW / 32)
// consecutive slots, a local pass plus a log-depth shuffle scan over the 32 lanes.
// Slot reuse: each call site owns a slot S (votes alternate between two ring slots), and
// every operation ends at a cluster barrier, so a slot is rewritten only after every
// warp of the cluster has read it.
#pragma once
#include "tv_comm.cuh"
#include "tv_cl_util.cuh"

namespace tvp {

template <typename T, int WPL, int NCTA>
struct CComm {
    static constexpr bool kCluster = true;
    static constexpr int NW = WPL * NCTA;            // warps holding the line
    static constexpr int Q = (NW + 31) / 32;         // slots per lane in the cross-warp combine
    static constexpr int M = 0x3fffffff, F = 1 << 30;
    int l;              // lane
    int w;              // warp within the line: rank * WPL + warp
    T* sv;              // [kCommSlots][3][NW]  (this CTA's copy)
    int* si;            // [kCommSlots][NW]
    int* sf;            // [2][NW] vote ring
    uint32_t sv_s, si_s, sf_s;   // shared::cta addresses (the same in every CTA)
    mutable int vr;     // vote ring position (line-uniform)

    __device__ __forceinline__ bool first_lane() const { return w == 0 && l == 0; }
    __device__ __forceinline__ T V(int s, int j, int ww) const { return sv[(s * 3 + j) * NW + ww]; }
    __device__ __forceinline__ int I(int s, int ww) const { return si[s * NW + ww]; }

    // The warp's value(s) from lane `src` into slot (s, w) of every CTA: lane d stores to CTA d.
    __device__ __forceinline__ void put1(int s, T v, int src) const {
        const T b = __shfl_sync(FULL, v, src);
        if (l < NCTA) cl_put(cl_map(sv_s + (uint32_t)(((s * 3) * NW + w) * sizeof(T)), l), b);
    }
    __device__ __forceinline__ void put2(int s, T v0, int src0, T v1, int src1) const {
        const T b0 = __shfl_sync(FULL, v0, src0), b1 = __shfl_sync(FULL, v1, src1);
        if (l < NCTA) {
            cl_put(cl_map(sv_s + (uint32_t)(((s * 3) * NW + w) * sizeof(T)), l), b0);
            cl_put(cl_map(sv_s + (uint32_t)(((s * 3 + 1) * NW + w) * sizeof(T)), l), b1);
        }
    }
    __device__ __forceinline__ void put3(int s, T v0, T v1, T v2, int src) const {
        const T b0 = __shfl_sync(FULL, v0, src), b1 = __shfl_sync(FULL, v1, src), b2 = __shfl_sync(FULL, v2, src);
        if (l < NCTA) {
            cl_put(cl_map(sv_s + (uint32_t)(((s * 3) * NW + w) * sizeof(T)), l), b0);
            cl_put(cl_map(sv_s + (uint32_t)(((s * 3 + 1) * NW + w) * sizeof(T)), l), b1);
            cl_put(cl_map(sv_s + (uint32_t)(((s * 3 + 2) * NW + w) * sizeof(T)), l), b2);
        }
    }
    __device__ __forceinline__ void puti(int s, int v, int src) const {
        const int b = __shfl_sync(FULL, v, src);
        if (l < NCTA) cl_put(cl_map(si_s + (uint32_t)((s * NW + w) * 4), l), b);
    }

    template <int S>
    __device__ __forceinline__ T prev(T v) const {
        T p = shup<32>(v, 1);
        put1(S, v, 31);
        cl_sync();
        if (l == 0 && w > 0) p = V(S, 0, w - 1);
        return first_lane() ? T(0) : p;
    }
    template <int S>
    __device__ __forceinline__ T next(T v) const {
        T nx = shdn<32>(v, 1);
        put1(S, v, 0);
        cl_sync();
        if (l == 31 && w + 1 < NW) nx = V(S, 0, w + 1);
        return nx;
    }
    template <int S>
    __device__ __forceinline__ void prev_next(T vp, T vn, T& p, T& nx) const {
        p = shup<32>(vp, 1);
        nx = shdn<32>(vn, 1);
        put2(S, vp, 31, vn, 0);
        cl_sync();
        if (l == 0 && w > 0) p = V(S, 0, w - 1);
        if (l == 31 && w + 1 < NW) nx = V(S, 1, w + 1);
        if (first_lane()) p = T(0);
    }

    // votes over the whole line (two ring slots alternate)
    __device__ __forceinline__ int vote_(int mine) const {
        const int slot = vr;
        vr ^= 1;
        if (l < NCTA) cl_put(cl_map(sf_s + (uint32_t)((slot * NW + w) * 4), l), mine);
        cl_sync();
        int acc = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            acc += (i < NW) ? sf[slot * NW + i] : 0;
        }
        return __reduce_add_sync(FULL, acc);
    }
    __device__ __forceinline__ bool any(bool p) const { return vote_(__any_sync(FULL, p) ? 1 : 0) != 0; }
    __device__ __forceinline__ bool all(bool p) const { return vote_(__all_sync(FULL, p) ? 1 : 0) == NW; }
    __device__ __forceinline__ bool uany(bool p) const { return p; }     // line-uniform already
    // bits set on every lane of the line (one vote)
    __device__ __forceinline__ uint32_t all_bits(uint32_t m) const {
        const int slot = vr;
        vr ^= 1;
        const uint32_t wm = __reduce_and_sync(FULL, m);
        if (l < NCTA) cl_put(cl_map(sf_s + (uint32_t)((slot * NW + w) * 4), l), (int)wm);
        cl_sync();
        uint32_t acc = 0xffffffffu;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            if (i < NW) acc &= (uint32_t)sf[slot * NW + i];
        }
        return __reduce_and_sync(FULL, acc);
    }

    // fixed-order sums: lane partials over its Q slots, then a fixed xor tree
    template <int S>
    __device__ __forceinline__ T sum(T v) const {
        v = group_sum<32>(v);
        put1(S, v, 0);
        cl_sync();
        T a = T(0);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            a += (i < NW) ? V(S, 0, i) : T(0);
        }
        return group_sum<32>(a);
    }
    template <int S>
    __device__ __forceinline__ void sum3(T& a, T& b, T& c) const {
        a = group_sum<32>(a);
        b = group_sum<32>(b);
        c = group_sum<32>(c);
        put3(S, a, b, c, 0);
        cl_sync();
        T xa = T(0), xb = T(0), xc = T(0);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            if (i < NW) { xa += V(S, 0, i); xb += V(S, 1, i); xc += V(S, 2, i); }
        }
        a = group_sum<32>(xa);
        b = group_sum<32>(xb);
        c = group_sum<32>(xc);
    }
    template <int S>
    __device__ __forceinline__ T max_(T v) const {
        v = group_max<32>(v);
        put1(S, v, 0);
        cl_sync();
        T a = V(S, 0, 0);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            if (i < NW) a = max(a, V(S, 0, i));
        }
        return group_max<32>(a);
    }

    // ---- segmented scans (same warp-level plan as Comm<T, 32, .>)
    using Seg = typename Comm<T, 32, 1>::Seg;
    __device__ __forceinline__ Seg seg_plan(bool f) const {
        const Comm<T, 32, 1> c1{l, 0, nullptr, nullptr};
        return c1.seg_plan(f);
    }

    // Exclusive segmented prefix over warps 0..w-1 of (a, c|flag) held in slot S
    // (c: count in bits 0..29, flag bit 30 = the warp holds a segment head).
    template <int S>
    __device__ __forceinline__ void warp_prefix_ac(T& ca, int& cc) const {
        T pa[Q];
        int pc[Q];
        T xa = T(0);
        int xc = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            const T ra = (i < NW) ? V(S, 0, i) : T(0);
            const int rc = (i < NW) ? I(S, i) : 0;
            if (rc & F) { xa = ra; xc = rc; } else { xa += ra; xc = ((xc & M) + (rc & M)) | (xc & F); }
            pa[q] = xa;
            pc[q] = xc;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shup<32>(xa, d);
            const int c2 = shup<32>(xc, d);
            if (l >= d && !(xc & F)) { xa += a2; xc = ((xc & M) + (c2 & M)) | (c2 & F); }
        }
        T la = shup<32>(xa, 1);
        int lc = shup<32>(xc, 1);
        if (l == 0) { la = T(0); lc = 0; }
        // inclusive value at slot w - 1
        const int i = w - 1, L = (i >= 0 ? i : 0) / Q, qq = (i >= 0 ? i : 0) - L * Q;
        T sa = pa[0];
        int sc = pc[0];
#pragma unroll
        for (int q = 1; q < Q; ++q)
            if (qq == q) { sa = pa[q]; sc = pc[q]; }
        T ia = (sc & F) ? sa : la + sa;
        int ic = (sc & F) ? sc : (((lc & M) + (sc & M)) | (lc & F));
        ia = __shfl_sync(FULL, ia, L);
        ic = __shfl_sync(FULL, ic, L);
        ca = (w > 0) ? ia : T(0);
        cc = (w > 0) ? (ic & M) : 0;
    }

    template <int S, int E>
    __device__ __forceinline__ void scan_fwd(const Seg& g, T& a, int& c) const {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shup<32>(a, d);
            if (d <= g.D) a += a2;
        }
        const int ch = __shfl_sync(FULL, c, g.h);
        const int ci = g.hh ? g.D * E + ch : (g.D + 1) * E;
        T ea = shup<32>(a, 1);
        int ecf = shup<32>(ci | (g.hh ? F : 0), 1);
        if (l == 0) { ea = T(0); ecf = 0; }
        const T a31 = __shfl_sync(FULL, a, 31);
        const int c31 = __shfl_sync(FULL, ci | (g.hh ? F : 0), 31);
        if (l < NCTA) {
            cl_put(cl_map(sv_s + (uint32_t)(((S * 3) * NW + w) * sizeof(T)), l), a31);
            cl_put(cl_map(si_s + (uint32_t)((S * NW + w) * 4), l), c31);
        }
        cl_sync();
        T ca;
        int cc;
        warp_prefix_ac<S>(ca, cc);
        if (!(ecf & F)) { ea += ca; ecf += cc; }
        a = ea;
        c = ecf & M;
    }

    template <int S>
    __device__ __forceinline__ void scan_fwd2(const Seg& g, T& a, T& b) const {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shup<32>(a, d), b2 = shup<32>(b, d);
            if (d <= g.D) { a += a2; b += b2; }
        }
        T ea = shup<32>(a, 1), eb = shup<32>(b, 1);
        if (l == 0) { ea = T(0); eb = T(0); }
        const T a31 = __shfl_sync(FULL, a, 31), b31 = __shfl_sync(FULL, b, 31);
        const int f31 = __shfl_sync(FULL, g.hh ? 1 : 0, 31);
        if (l < NCTA) {
            cl_put(cl_map(sv_s + (uint32_t)(((S * 3) * NW + w) * sizeof(T)), l), a31);
            cl_put(cl_map(sv_s + (uint32_t)(((S * 3 + 1) * NW + w) * sizeof(T)), l), b31);
            cl_put(cl_map(si_s + (uint32_t)((S * NW + w) * 4), l), f31);
        }
        cl_sync();
        // exclusive segmented prefix of (a, b) over warps 0..w-1, flag = warp holds a head
        T pa[Q], pb[Q];
        int pf[Q];
        T xa = T(0), xb = T(0);
        int xf = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int i = l * Q + q;
            const T ra = (i < NW) ? V(S, 0, i) : T(0), rb = (i < NW) ? V(S, 1, i) : T(0);
            const int rf = (i < NW) ? I(S, i) : 0;
            if (rf) { xa = ra; xb = rb; xf = 1; } else { xa += ra; xb += rb; }
            pa[q] = xa; pb[q] = xb; pf[q] = xf;
        }
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T a2 = shup<32>(xa, d), b2 = shup<32>(xb, d);
            const int f2 = shup<32>(xf, d);
            if (l >= d && !xf) { xa += a2; xb += b2; xf = f2; }
        }
        T la = shup<32>(xa, 1), lb = shup<32>(xb, 1);
        if (l == 0) { la = T(0); lb = T(0); }
        const int i = w - 1, L = (i >= 0 ? i : 0) / Q, qq = (i >= 0 ? i : 0) - L * Q;
        T sa = pa[0], sb = pb[0];
        int sfl = pf[0];
#pragma unroll
        for (int q = 1; q < Q; ++q)
            if (qq == q) { sa = pa[q]; sb = pb[q]; sfl = pf[q]; }
        T ia = sfl ? sa : la + sa, ib = sfl ? sb : lb + sb;
        ia = __shfl_sync(FULL, ia, L);
        ib = __shfl_sync(FULL, ib, L);
        if (w > 0 && !g.hx) { ea += ia; eb += ib; }
        a = ea;
        b = eb;
    }

    // Value of the nearest flagged line lane strictly to the right (0 if none).
    template <int S>
    __device__ __forceinline__ T scan_rev(const Seg& g, T v) const {
        T e = __shfl_sync(FULL, v, g.rs);
        if (!g.rf) e = T(0);
        const T vf = __shfl_sync(FULL, v, g.fm ? __ffs(g.fm) - 1 : 0);
        if (l < NCTA) {
            cl_put(cl_map(sv_s + (uint32_t)(((S * 3) * NW + w) * sizeof(T)), l), vf);
            cl_put(cl_map(si_s + (uint32_t)((S * NW + w) * 4), l), g.fm != 0u ? 1 : 0);
        }
        cl_sync();
        // suffix: nearest flagged slot at or right of each slot
        T sv_[Q];
        int sf_[Q];
        T cur = T(0);
        int has = 0;
#pragma unroll
        for (int q = Q - 1; q >= 0; --q) {
            const int i = l * Q + q;
            if (i < NW && I(S, i)) { cur = V(S, 0, i); has = 1; }
            sv_[q] = cur;
            sf_[q] = has;
        }
        T xv = cur;
        int xf = has;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T v2 = shdn<32>(xv, d);
            const int f2 = shdn<32>(xf, d);
            if (l + d < 32 && !xf) { xv = v2; xf = f2; }
        }
        T rv = shdn<32>(xv, 1);
        int rf = shdn<32>(xf, 1);
        if (l == 31) { rv = T(0); rf = 0; }
        const int i = w + 1, L = (i < NW ? i : 0) / Q, qq = (i < NW ? i : 0) - L * Q;
        T sa = sv_[0];
        int sfl = sf_[0];
#pragma unroll
        for (int q = 1; q < Q; ++q)
            if (qq == q) { sa = sv_[q]; sfl = sf_[q]; }
        T r = sfl ? sa : (rf ? rv : T(0));
        r = __shfl_sync(FULL, r, L);
        if (!g.rf && w + 1 < NW) e = r;
        return e;
    }
};

}  // namespace tvp
