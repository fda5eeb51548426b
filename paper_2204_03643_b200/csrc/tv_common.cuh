// tv_common.cuh -- shared device helpers of the sm_100a TV-prox kernels.
//
// Line layout used by every kernel: a "line" (1D row, 2D row or 2D column) of
// n <= LPR*E samples is held by a group of LPR consecutive lanes of a warp;
// lane l of the group holds the CONTIGUOUS samples i = l*E + k, k = 0..E-1,
// in registers.  Edge i (between samples i and i+1) belongs to the lane that
// holds sample i.  Edges i >= n-1 (and edges with lam_i = 0) are "pinned":
// their dual is fixed at 0, which isolates the padding samples.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvp {

constexpr unsigned FULL = 0xffffffffu;

template <typename T> struct Num;
template <> struct Num<float> {
    static constexpr float eps = 5.9604645e-08f;   // 2^-24, unit roundoff
    static constexpr int max_iters = 64;
};
template <> struct Num<double> {
    static constexpr double eps = 1.1102230246251565e-16;  // 2^-53
    static constexpr int max_iters = 100;
};

// Padded shared-memory index: one spare word every 32 so that lane l reading
// sample l*E + k hits distinct banks (E a multiple of 32 or odd).
__device__ __forceinline__ int spad(int i) { return i + (i >> 5); }
__host__ __device__ constexpr int spad_len(int m) { return m + (m >> 5) + 1; }

template <int W, typename T>
__device__ __forceinline__ T shup(T v, int d) { return __shfl_up_sync(FULL, v, d, W); }
template <int W, typename T>
__device__ __forceinline__ T shdn(T v, int d) { return __shfl_down_sync(FULL, v, d, W); }
template <int W, typename T>
__device__ __forceinline__ T shxor(T v, int m) { return __shfl_xor_sync(FULL, v, m, W); }

template <int W, typename T>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
    for (int m = W / 2; m >= 1; m >>= 1) v += shxor<W>(v, m);
    return v;
}
template <int W, typename T>
__device__ __forceinline__ T group_max(T v) {
#pragma unroll
    for (int m = W / 2; m >= 1; m >>= 1) v = max(v, shxor<W>(v, m));
    return v;
}

// Group-wide vote: true iff pred holds on every lane of this lane's group.
template <int W>
__device__ __forceinline__ bool group_all(bool pred) {
    unsigned b = __ballot_sync(FULL, !pred);
    if (W == 32) return b == 0;
    unsigned lane = threadIdx.x & 31;
    unsigned gm = ((1u << W) - 1u) << (lane & ~(W - 1));
    return (b & gm) == 0;
}
template <int W>
__device__ __forceinline__ bool group_any(bool pred) { return !group_all<W>(!pred); }

// Reciprocal of a small positive count.  fp32: MUFU.RCP (<= 1 ulp), fp64: IEEE.
__device__ __forceinline__ float rcp_(float c) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(c));   // c >= 1 (a count): never subnormal
    return r;
}
__device__ __forceinline__ double rcp_(double c) { return 1.0 / c; }
// Division by a small positive count.  fp32: MUFU reciprocal (<= 2 ulp).
__device__ __forceinline__ float div_count(float a, int c) { return __fdividef(a, (float)c); }
__device__ __forceinline__ double div_count(double a, int c) { return a / (double)c; }

__device__ __forceinline__ float clampv(float v, float lo, float hi) { return fminf(fmaxf(v, lo), hi); }
__device__ __forceinline__ double clampv(double v, double lo, double hi) { return fmin(fmax(v, lo), hi); }

template <typename T> __device__ __forceinline__ bool finite_(T v) { return isfinite(v); }

template <typename T> __device__ __forceinline__ T nan_();
template <> __device__ __forceinline__ float nan_<float>() { return __int_as_float(0x7fc00000); }
template <> __device__ __forceinline__ double nan_<double>() { return __longlong_as_double(0x7ff8000000000000ll); }

// 2-bit edge codes of the saved mask (include/tvprox.h).
enum : uint32_t { CODE_FUSED = 0u, CODE_UP = 1u, CODE_DOWN = 2u, CODE_BOUNDARY = 3u };

template <typename T>
__device__ __forceinline__ uint32_t edge_code(T xl, T xr, bool lam_zero) {
    return xr > xl ? CODE_UP : (xr < xl ? CODE_DOWN : (lam_zero ? CODE_BOUNDARY : CODE_FUSED));
}

// Spread bits 0..15 of x to the even positions 0, 2, ..., 30 (inverse of compact_even).
__device__ __forceinline__ uint32_t spread_even(uint32_t x) {
    x &= 0x0000ffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// 2-bit codes of a lane's E <= 16 edges e0 .. e0 + E - 1 (edge k between samples k and
// k + 1 of the lane, x_r of the last one from the next lane), bit-parallel: jump bits,
// masked to the line's edges (< nedge), spread to codes at bits 2k; boundary code where
// lam = 0 and the values are equal.  Same codes as edge_code per edge.
// up / dn return the lanes' jump bits (edges coded CODE_UP / CODE_DOWN).
template <typename T, int E>
__device__ __forceinline__ uint32_t lane_codes(const T (&w)[E], T wnext, int e0, int nedge, bool lam_zero,
                                               uint32_t& up, uint32_t& dn) {
    static_assert(E <= 16, "one word of codes per lane");
    up = 0u;
    dn = 0u;
#pragma unroll
    for (int k = 0; k < E; ++k) {
        const T xr = (k + 1 < E) ? w[(k + 1 < E) ? k + 1 : k] : wnext;
        up |= (xr > w[k] ? 1u : 0u) << k;
        dn |= (xr < w[k] ? 1u : 0u) << k;
    }
    constexpr uint32_t allm = (E == 32) ? 0xffffffffu : ((1u << (E & 31)) - 1u);
    const int ne = nedge - e0;
    const uint32_t vm = ne >= E ? allm : (ne <= 0 ? 0u : ((1u << ne) - 1u));
    up &= vm;
    dn &= vm;
    const uint32_t bz = lam_zero ? (vm & ~(up | dn)) : 0u;
    return spread_even(up | bz) | (spread_even(dn | bz) << 1);
}
template <typename T, int E>
__device__ __forceinline__ uint32_t lane_codes(const T (&w)[E], T wnext, int e0, int nedge, bool lam_zero) {
    uint32_t up, dn;
    return lane_codes<T, E>(w, wnext, e0, nedge, lam_zero, up, dn);
}

// Gather the even bits of x (bits 0, 2, ..., 30) into bits 0..15.
__device__ __forceinline__ uint32_t compact_even(uint32_t x) {
    x &= 0x55555555u;
    x = (x | (x >> 1)) & 0x33333333u;
    x = (x | (x >> 2)) & 0x0f0f0f0fu;
    x = (x | (x >> 4)) & 0x00ff00ffu;
    x = (x | (x >> 8)) & 0x0000ffffu;
    return x;
}

// Extract the 2E-bit window of mask codes for edges [e0, e0+E) of one line
// (word array `mw`, nw words).  Returns per-edge bitmasks: bnd = code != 0,
// neg = code == DOWN, pos = code == UP (bit-parallel: lo/hi code bits, then
// even-bit compaction, 16 edges per step).  Split into the word loads
// (mask_words_ld, issued early to overlap their latency) and the decode.
template <int E> struct MaskWin {
    static constexpr int NS = (2 * E + 31) / 32;   // words of the aligned window
    uint32_t w[NS + 1];
};

template <int E>
__device__ __forceinline__ void mask_words_ld(const uint32_t* __restrict__ mw, int nw, int e0, MaskWin<E>& mwin) {
    const int w0 = e0 >> 4;
#pragma unroll
    for (int j = 0; j <= MaskWin<E>::NS; ++j) mwin.w[j] = (w0 + j < nw) ? __ldg(mw + w0 + j) : 0u;
}

template <int E>
__device__ __forceinline__ void mask_decode(const MaskWin<E>& mwin, int e0, uint32_t& bnd, uint32_t& pos,
                                            uint32_t& neg) {
    const int sh = (e0 & 15) * 2;
    bnd = pos = neg = 0;
#pragma unroll
    for (int j = 0; j < MaskWin<E>::NS; ++j) {
        const uint32_t c = __funnelshift_r(mwin.w[j], mwin.w[j + 1], sh);   // 16 codes
        const uint32_t lo = compact_even(c), hi = compact_even(c >> 1);
        bnd |= (lo | hi) << (16 * j);
        pos |= (lo & ~hi) << (16 * j);
        neg |= (hi & ~lo) << (16 * j);
    }
    constexpr uint32_t m = (E >= 32) ? 0xffffffffu : ((1u << (E & 31)) - 1u);
    bnd &= m; pos &= m; neg &= m;
}

// Bits k of an E-edge lane window with k >= nv (edges past the line end, pinned).
template <int E>
__device__ __forceinline__ uint32_t pin_tail(int nv) {
    constexpr uint32_t all = (E >= 32) ? 0xffffffffu : ((1u << (E & 31)) - 1u);
    if (nv <= 0) return all;
    if (nv >= E) return 0u;
    return all & ~((1u << nv) - 1u);
}

template <int E>
__device__ __forceinline__ void mask_window(const uint32_t* __restrict__ mw, int nw, int e0,
                                            uint32_t& bnd, uint32_t& pos, uint32_t& neg) {
    MaskWin<E> mwin;
    mask_words_ld<E>(mw, nw, e0, mwin);
    mask_decode<E>(mwin, e0, bnd, pos, neg);
}

}  // namespace tvp
