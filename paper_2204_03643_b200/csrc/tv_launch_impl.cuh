// tv_launch_impl.cuh -- launcher templates (included once per dtype unit).
#pragma once
#include <atomic>
#include <algorithm>
#include <mutex>
#include <unordered_map>
#include <cstdlib>
#include <cstdio>

#include "tv_kernels.cuh"
#include "tv_cluster.cuh"
#include "tv_long.cuh"
#include "tv_launch.h"

namespace tvp {

// Persistent grid: min(work, SMs x resident blocks per SM) for this kernel on the
// current device.  The dynamic shared-memory opt-in and the occupancy query are per
// (device, kernel, smem) -- the attribute belongs to the device context -- and cached
// under a mutex; a failed opt-in (more shared memory than the device allows) is
// returned as an error instead of launching.
struct OccKey {
    int dev;
    const void* fn;
    size_t smem;
    bool operator==(const OccKey& o) const { return dev == o.dev && fn == o.fn && smem == o.smem; }
};
struct OccKeyHash {
    size_t operator()(const OccKey& k) const {
        return std::hash<const void*>()(k.fn) ^ (std::hash<size_t>()(k.smem) * 31u) ^ ((size_t)k.dev << 48);
    }
};
template <typename K>
static cudaError_t persistent_grid(K kern, int threads, size_t smem, int64_t work_blocks, int& grid) {
    static std::mutex mu;
    static std::unordered_map<OccKey, int, OccKeyHash> occ_cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int sms = 148;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    int occ = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        const OccKey key{dev, reinterpret_cast<const void*>(kern), smem};
        auto it = occ_cache.find(key);
        if (it == occ_cache.end()) {
            if (smem > 48 * 1024) {
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
            }
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
            if (e != cudaSuccess) return e;
            occ_cache[key] = occ;
        } else {
            occ = it->second;
        }
    }
    if (occ < 1) return cudaErrorInvalidConfiguration;   // does not fit one SM
    int64_t g = std::min<int64_t>(work_blocks, (int64_t)sms * occ);
    grid = (int)std::max<int64_t>(g, 1);
    return cudaSuccess;
}

// Environment knobs of the A/B tuning builds: read once per process (thread-safe
// function-local statics), never mutated afterwards.
static int env_int(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

#define TVP_GEO_DISPATCH(n, ...)                                               \
    do {                                                                       \
        Geo g_ = pick_geo(n, (int)sizeof(T));                                  \
        if (g_.LPR == 16) {                                                    \
            if constexpr (sizeof(T) == 4) {                                    \
                if (g_.E == 14) { constexpr int E_ = 14, L_ = 16; __VA_ARGS__; }   \
                else { constexpr int E_ = 8, L_ = 16; __VA_ARGS__; }           \
            }                                                                  \
        } else if (g_.LPR == 8) {                                              \
            switch (g_.E) {                                                    \
                case 2: { constexpr int E_ = 2, L_ = 8; __VA_ARGS__; } break;         \
                case 4: { constexpr int E_ = 4, L_ = 8; __VA_ARGS__; } break;         \
                case 7: { constexpr int E_ = 7, L_ = 8; __VA_ARGS__; } break;         \
                default: { constexpr int E_ = 8, L_ = 8; __VA_ARGS__; } break;        \
            }                                                                  \
        } else {                                                               \
            switch (g_.E) {                                                    \
                case 4: { constexpr int E_ = 4, L_ = 32; __VA_ARGS__; } break;        \
                case 7: { constexpr int E_ = 7, L_ = 32; __VA_ARGS__; } break;        \
                case 8: { constexpr int E_ = 8, L_ = 32; __VA_ARGS__; } break;        \
                case 16: { constexpr int E_ = 16, L_ = 32; __VA_ARGS__; } break;      \
                default: { constexpr int E_ = 32, L_ = 32; __VA_ARGS__; } break;      \
            }                                                                  \
        }                                                                      \
    } while (0)

constexpr int kRowWPB = 4;

// 513..1024-sample row-forward lines always take two warps per line (k_row_fwd_w, E = 16).
// (The former A/B knob TVP_ROW_SPLIT=0 sent them to the staged one-warp kernel, whose
// warp mask-word buffer holds 32 words -- lines of <= 512 samples -- and overran it.)
static int row_fwd_split() { return 2; }
// Warps per column-tile CTA (tile = WPB x 32 / LPR lines, x2 for one-warp lines), per
// kernel and geometry from same-box A/B runs: fp32 one-warp
// E = 16 column solves and adjoints (C4) 4 warps (adjoint: C4 bwd 0.441 -> 0.434 ms vs 8;
// 2 warps 0.449), E = 14 column adjoints (C5) 4 warps, otherwise 8.
// TVP_COL_WPB forces one value for every column kernel (A/B builds).
// fp64 lines of E = 32 (513..1024 samples) use 4 warps (8 columns): 8 would need
// 2 x 16 x 1055 x 8 B = 270 KB of shared memory, above the 227 KB per-CTA limit.
#ifndef TVP_COLF14_WPB
#define TVP_COLF14_WPB 8
#endif
template <typename T, int E, int LPR> constexpr int col_wpb_fwd() {
#ifdef TVP_COL_WPB
    return TVP_COL_WPB;
#else
    return (sizeof(T) == 4 && E == 14) ? TVP_COLF14_WPB
         : (((sizeof(T) == 4 && E == 16 && LPR == 32) || (sizeof(T) == 8 && E == 32)) ? 4 : 8);
#endif
}
#ifndef TVP_COLB14_WPB
#define TVP_COLB14_WPB 4
#endif
#ifndef TVP_COLB16_WPB
#define TVP_COLB16_WPB 4
#endif
template <typename T, int E, int LPR> constexpr int col_wpb_bwd() {
#ifdef TVP_COL_WPB
    return TVP_COL_WPB;
#else
    return (sizeof(T) == 4 && E == 14) ? TVP_COLB14_WPB
         : ((sizeof(T) == 4 && E == 16 && LPR == 32) ? TVP_COLB16_WPB : ((sizeof(T) == 8 && E == 32) ? 4 : 8));
#endif
}

// TVP_COARSE16=0 (A/B): half-warp lines (LPR = 16) solve cold without the coarse start.
static bool coarse16_knob() {
    static const bool v = env_int("TVP_COARSE16", 1) != 0;
    return v;
}

// TVP_ROW_DIRECT=0 (A/B): rows of <= 512 samples staged through shared memory (k_row_fwd /
// k_row_bwd) instead of the register-direct kernels (k_row_fwd_r / k_row_bwd_r).
static bool row_direct_knob() {
    static const bool v = env_int("TVP_ROW_DIRECT", 1) != 0;
    return v;
}

template <typename T, int E, int LPR, bool PE, bool DYK, bool LSP>
static cudaError_t row_fwd_t(RowFwdArgs<T> a, cudaStream_t s) {
    constexpr int G = 32 / LPR;
    if (LPR < 32 && !coarse16_knob()) a.coarse = 0;
    if (row_direct_knob()) {
        auto kern = k_row_fwd_r<T, E, LPR, PE, DYK, kRowWPB, LSP>;
        const int64_t groups = (a.nlines + G - 1) / G;
        int grid = 0;
        cudaError_t e = persistent_grid(kern, kRowWPB * 32, 0, (groups + kRowWPB - 1) / kRowWPB, grid);
        if (e != cudaSuccess) return e;
        kern<<<grid, kRowWPB * 32, 0, s>>>(a);
        count_launch();
        return cudaGetLastError();
    }
    constexpr int LP = line_pitch<E, LPR>();
    const size_t smem = (size_t)kRowWPB * (DYK ? 2 : 1) * G * LP * sizeof(T) + (size_t)kRowWPB * 32 * 4;
    auto kern = k_row_fwd<T, E, LPR, PE, DYK, kRowWPB, LSP>;
    const int64_t groups = (a.nlines + G - 1) / G;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, kRowWPB * 32, smem, (groups + kRowWPB - 1) / kRowWPB, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, kRowWPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T, int E, int WPL, bool PE, bool DYK, bool LSP>
static cudaError_t row_fwd_w_t(const RowFwdArgs<T>& a, cudaStream_t s) {
    auto kern = k_row_fwd_w<T, E, WPL, PE, DYK, LSP>;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPL * 32, 0, a.nlines, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPL * 32, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

// TVP_COARSE=0 disables the coarse initial bound set of cold solves (A/B only).
static bool coarse_knob() {
    static const bool v = env_int("TVP_COARSE", 1) != 0;
    return v;
}

// Coarse pre-pass for the long-row geometry (E = 16 fine blocks): writes the initial
// mask into mask_out, which the fine kernel then reads as its warm start.
template <typename T, int EF, int CPL, bool DYK>
static cudaError_t coarse_rows_t(const RowFwdArgs<T>& a, cudaStream_t s) {
    constexpr int WPB = 4;
    auto kern = k_coarse_rows<T, EF, CPL, DYK, WPB>;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, 0, (a.nlines + WPB - 1) / WPB, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T, bool DYK>
static cudaError_t coarse_rows2_t(const RowFwdArgs<T>& a, cudaStream_t s) {
    constexpr int WPB = 4;
    static const bool four = env_int("TVP_COARSE4", 1) != 0;   // four lines per warp (A/B knob)
    if (four) {
        auto kern4 = k_coarse_rows4<T, DYK, WPB>;
        const int64_t quads = (a.nlines + 3) / 4;
        int grid = 0;
        cudaError_t e = persistent_grid(kern4, WPB * 32, 0, (quads + WPB - 1) / WPB, grid);
        if (e != cudaSuccess) return e;
        kern4<<<grid, WPB * 32, 0, s>>>(a);
        count_launch();
        return cudaGetLastError();
    }
    auto kern = k_coarse_rows2<T, DYK, WPB>;
    const int64_t pairs = (a.nlines + 1) / 2;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, 0, (pairs + WPB - 1) / WPB, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

// TVP_COARSE_PASS=0 keeps the coarse solve inside the fine forward kernel (A/B); the
// default runs it as a pre-pass (two lines per warp for 513..1024-sample lines).
static int coarse_pass_knob() {
    static const int v = env_int("TVP_COARSE_PASS", 2);
    return v;
}

// Row-forward set-up shared by both line-search flavours: the coarse initial bound set
// of cold solves (reading O7) -- in-kernel (a.coarse = 1) or, for the E = 16 fine
// geometries, as a separate pre-pass kernel that writes the initial mask into
// mask_out, which the fine kernel then reads as its warm start (a.mask_in).
template <typename T>
cudaError_t row_fwd_prepass(RowFwdArgs<T>& a, bool per_edge, bool dykstra, cudaStream_t s) {
    a.coarse = (a.mask_in == nullptr && !per_edge && coarse_knob()) ? 1 : 0;
    if (a.n > 1024) {
        if (TVP_COARSE_MAXWPL < 4) a.coarse = 0;   // long rows: in-kernel coarse solve
        return cudaSuccess;
    }
    if (!(a.coarse && a.mask_out && a.n >= 3 * 4 && coarse_pass_knob())) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    if (a.n > 512 && row_fwd_split() == 2) {
        e = dykstra ? coarse_rows2_t<T, true>(a, s) : coarse_rows2_t<T, false>(a, s);
    } else if (a.n > 256 && a.n <= 512 && pick_geo(a.n).E == 16) {
        // (E <= 8 geometries keep the in-kernel coarse solve: their short loops do not
        // spill the I-cache, and a separate pass measured slower at C5)
        e = dykstra ? coarse_rows_t<T, 16, 1, true>(a, s) : coarse_rows_t<T, 16, 1, false>(a, s);
    } else {
        return cudaSuccess;
    }
    if (e != cudaSuccess) return e;
    a.mask_in = a.mask_out;                      // in place: each line reads its words before writing them
    a.coarse = 0;
    return cudaSuccess;
}

// f4 beyond one CTA: a thread-block cluster per row (tv_long.cuh), defined below.
constexpr int64_t long_row_per_cta(int esz) { return esz == 4 ? 16 * 32 * 16 : 16 * 32 * 8; }
template <typename T, bool LSP> cudaError_t launch_row_fwd_long(const RowFwdArgs<T>& a, bool per_edge, cudaStream_t s);
template <typename T> cudaError_t launch_row_bwd_long(const RowBwdArgs<T>& a, bool per_edge, cudaStream_t s);

template <typename T, bool LSP>
cudaError_t launch_row_fwd_ls(RowFwdArgs<T> a, bool per_edge, bool dykstra, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (a.n > long_row_per_cta((int)sizeof(T))) return launch_row_fwd_long<T, LSP>(a, per_edge, s);
    if (a.n > 1024) {
        // long 1D rows (f4): one CTA of WPL warps holds the row in registers, E = 16
        // (fp32) / 8 (fp64) samples per lane; in-kernel coarse solve
        if constexpr (sizeof(T) == 4) {
            if (a.n <= 2048) return per_edge ? row_fwd_w_t<T, 16, 4, true, false, LSP>(a, s) : row_fwd_w_t<T, 16, 4, false, false, LSP>(a, s);
            if (a.n <= 4096) return per_edge ? row_fwd_w_t<T, 16, 8, true, false, LSP>(a, s) : row_fwd_w_t<T, 16, 8, false, false, LSP>(a, s);
            return per_edge ? row_fwd_w_t<T, 16, 16, true, false, LSP>(a, s) : row_fwd_w_t<T, 16, 16, false, false, LSP>(a, s);
        } else {
            if (a.n <= 2048) return per_edge ? row_fwd_w_t<T, 8, 8, true, false, LSP>(a, s) : row_fwd_w_t<T, 8, 8, false, false, LSP>(a, s);
            return per_edge ? row_fwd_w_t<T, 8, 16, true, false, LSP>(a, s) : row_fwd_w_t<T, 8, 16, false, false, LSP>(a, s);
        }
    }
    if (a.n > 512 && row_fwd_split() == 2) {     // 1024-sample lines: two warps x 16 samples per lane
        if (dykstra) return row_fwd_w_t<T, 16, 2, false, true, LSP>(a, s);
        if (per_edge) return row_fwd_w_t<T, 16, 2, true, false, LSP>(a, s);
        return row_fwd_w_t<T, 16, 2, false, false, LSP>(a, s);
    }
    TVP_GEO_DISPATCH(a.n, {
        if (dykstra) e = row_fwd_t<T, E_, L_, false, true, LSP>(a, s);
        else if (per_edge) e = row_fwd_t<T, E_, L_, true, false, LSP>(a, s);
        else e = row_fwd_t<T, E_, L_, false, false, LSP>(a, s);
    });
    return e;
}

template <int WPB, int LPR> constexpr int col_tile() { return WPB * (32 / LPR) * (LPR == 32 ? 2 : 1); }
template <typename T, int E, int WPB, int LPR> constexpr int col_tile_fwd() { return col_tile<WPB, LPR>() * colf_tm<T, E>(); }

template <typename T, int E, int LPR, bool LSP>
static cudaError_t col_fwd_t(ColFwdArgs<T> a, cudaStream_t s) {
    constexpr int WPB = col_wpb_fwd<T, E, LPR>();
    constexpr int LP = line_pitch<E, LPR>();
    constexpr int TC = col_tile_fwd<T, E, WPB, LPR>();
    a.TC = TC;
    if (LPR < 32 && !coarse16_knob()) a.coarse = 0;
    const size_t smem = (size_t)2 * TC * LP * sizeof(T) + (size_t)WPB * 64 * 4;
    auto kern = k_col_fwd<T, E, LPR, WPB, LSP>;
    const int64_t tiles = a.planes * ((a.W + TC - 1) / TC);
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, smem, tiles, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T, bool LSP>
cudaError_t launch_col_fwd_ls(ColFwdArgs<T> a, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    a.coarse = (a.mask_in == nullptr && coarse_knob()) ? 1 : 0;
    TVP_GEO_DISPATCH(a.H, { e = col_fwd_t<T, E_, L_, LSP>(a, s); });
    return e;
}

template <typename T, int E, int LPR, bool DYK, bool PE>
static cudaError_t row_bwd_t(const RowBwdArgs<T>& a, cudaStream_t s) {
    constexpr int G = 32 / LPR;
    if (row_direct_knob()) {
        auto kern = k_row_bwd_r<T, E, LPR, DYK, PE, kRowWPB>;
        const int64_t groups = (a.nlines + G - 1) / G;
        int grid = 0;
        cudaError_t e = persistent_grid(kern, kRowWPB * 32, 0, (groups + kRowWPB - 1) / kRowWPB, grid);
        if (e != cudaSuccess) return e;
        kern<<<grid, kRowWPB * 32, 0, s>>>(a);
        count_launch();
        return cudaGetLastError();
    }
    constexpr int LP = line_pitch<E, LPR>();
    const size_t smem = (size_t)kRowWPB * (DYK ? 2 : 1) * G * LP * sizeof(T);
    auto kern = k_row_bwd<T, E, LPR, DYK, PE, kRowWPB>;
    const int64_t groups = (a.nlines + G - 1) / G;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, kRowWPB * 32, smem, (groups + kRowWPB - 1) / kRowWPB, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, kRowWPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T, int E, int WPL, bool DYK, bool PE>
static cudaError_t row_bwd_w_t(const RowBwdArgs<T>& a, cudaStream_t s) {
    auto kern = k_row_bwd_w<T, E, WPL, DYK, PE>;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPL * 32, 0, a.nlines, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPL * 32, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_row_bwd(const RowBwdArgs<T>& a, bool dykstra, bool per_edge, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (a.n > long_row_per_cta((int)sizeof(T))) return launch_row_bwd_long<T>(a, per_edge, s);
    if (a.n > 1024) {                             // long 1D rows (f4): one CTA of WPL warps per row
        if constexpr (sizeof(T) == 4) {
            if (a.n <= 2048) return per_edge ? row_bwd_w_t<T, 16, 4, false, true>(a, s) : row_bwd_w_t<T, 16, 4, false, false>(a, s);
            if (a.n <= 4096) return per_edge ? row_bwd_w_t<T, 16, 8, false, true>(a, s) : row_bwd_w_t<T, 16, 8, false, false>(a, s);
            return per_edge ? row_bwd_w_t<T, 16, 16, false, true>(a, s) : row_bwd_w_t<T, 16, 16, false, false>(a, s);
        } else {
            if (a.n <= 2048) return per_edge ? row_bwd_w_t<T, 8, 8, false, true>(a, s) : row_bwd_w_t<T, 8, 8, false, false>(a, s);
            return per_edge ? row_bwd_w_t<T, 8, 16, false, true>(a, s) : row_bwd_w_t<T, 8, 16, false, false>(a, s);
        }
    }
    if (a.n > 512) {                              // 2 warps x 16 samples per thread (same-box A/B best)
        if (dykstra) return row_bwd_w_t<T, 16, 2, true, false>(a, s);
        if (per_edge) return row_bwd_w_t<T, 16, 2, false, true>(a, s);
        return row_bwd_w_t<T, 16, 2, false, false>(a, s);
    }
    if (a.n > 256) {                              // 2 warps x 8
        if (dykstra) return row_bwd_w_t<T, 8, 2, true, false>(a, s);
        if (per_edge) return row_bwd_w_t<T, 8, 2, false, true>(a, s);
        return row_bwd_w_t<T, 8, 2, false, false>(a, s);
    }
    TVP_GEO_DISPATCH(a.n, {
        if (dykstra) e = row_bwd_t<T, E_, L_, true, false>(a, s);
        else if (per_edge) e = row_bwd_t<T, E_, L_, false, true>(a, s);
        else e = row_bwd_t<T, E_, L_, false, false>(a, s);
    });
    return e;
}

template <typename T, int E, int LPR>
static cudaError_t col_bwd_t(ColBwdArgs<T> a, cudaStream_t s) {
    constexpr int LP = line_pitch<E, LPR>();
    constexpr int WPB = col_wpb_bwd<T, E, LPR>();
    constexpr int TC = col_tile<WPB, LPR>();
    a.TC = TC;
    const size_t smem = (size_t)2 * TC * LP * sizeof(T);
    auto kern = k_col_bwd<T, E, LPR, WPB>;
    const int64_t tiles = a.planes * ((a.W + TC - 1) / TC);
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, smem, tiles, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_col_bwd(ColBwdArgs<T> a, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    TVP_GEO_DISPATCH(a.H, { e = col_bwd_t<T, E_, L_>(a, s); });
    return e;
}

template <typename T>
cudaError_t launch_lam_reduce(const LamReduceArgs<T>& a, cudaStream_t s) {
    if (a.nout <= 0) return cudaSuccess;
    dim3 g1((unsigned)a.nout, a.nchunk);
    k_lam_reduce1<T><<<g1, 256, 0, s>>>(a);
    count_launch();
    int g2 = (int)std::min<int64_t>(a.nout, 4096);
    k_lam_reduce2<T><<<g2, 256, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

static int elementwise_grid(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}
template <typename T>
cudaError_t launch_softplus(const T* t, T* lam, const T* g, T* gt, int64_t n, bool bwd, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (bwd) k_softplus_bwd<T><<<elementwise_grid(n), 256, 0, s>>>(t, g, gt, n);
    else k_softplus_fwd<T><<<elementwise_grid(n), 256, 0, s>>>(t, lam, n);
    count_launch();
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_axpby(const T* x, T* y, T a, T b, int64_t n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    k_axpby<T><<<elementwise_grid(n), 256, 0, s>>>(x, y, a, b, n);
    count_launch();
    return cudaGetLastError();
}

// Shared-memory row pitch of the fused plane kernels' [H][pitch] planes.  A warp reads 4 lines
// x 8 lanes: row pass lanes (g, l) at (4t + g, ER l + q), column pass at (EC l + q, 4t + g).
// For fp32 the pitch in [W, W + 32) with the fewest bank conflicts over both patterns (max
// ways, then total) is chosen once per (H, W); e.g. C3's 56 x 56 planes get pitch 56 (row
// reads 2-way, column reads conflict-free) instead of the odd pitch 57 (4-way / 2-way).
// fp64 keeps the odd pitch.
inline int plane_conflicts(int P, int ER, int EC, int H, int W, int& sum) {
    int worst = 0;
    sum = 0;
    for (int o = 0; o < 2; ++o) {
        const int E = o ? EC : ER, nl = o ? W : H, ne = o ? H : W;
        int wo = 0;
        for (int t = 0; t < (nl + 3) / 4 && t < 8; ++t)        // the bank pattern repeats in t with period 8
            for (int q = 0; q < E; ++q) {
                int cnt[32] = {0};
                for (int g = 0; g < 4; ++g)
                    for (int l = 0; l < 8; ++l) {
                        const int line = 4 * t + g, e = E * l + q;
                        if (line >= nl || e >= ne) continue;
                        const int h = o ? e : line, c = o ? line : e;
                        const int b = (h * P + c) & 31;
                        if (++cnt[b] > wo) wo = cnt[b];
                    }
            }
        worst = wo > worst ? wo : worst;
        sum += wo;
    }
    return worst;
}
template <typename T>
inline int plane_pitch(int H, int W, int ER, int EC) {
    if (sizeof(T) != 4 || H < 1 || H > 64 || W < 1 || W > 64) return W | 1;
    static std::atomic<int> cache[2][2][65][65];       // [ER==8][EC==8][H][W], 0 = not computed
    std::atomic<int>& c = cache[ER == 8][EC == 8][H][W];
    int v = c.load(std::memory_order_relaxed);
    if (v == 0) {
        int bw = 1 << 30, bs = 1 << 30;
        v = W | 1;
        for (int P = W; P < W + 32; ++P) {
            int sum;
            const int wv = plane_conflicts(P, ER, EC, H, W, sum);
            if (wv < bw || (wv == bw && sum < bs)) { v = P; bw = wv; bs = sum; }
        }
        c.store(v, std::memory_order_relaxed);         // idempotent: racing callers store the same value
    }
    return v;
}

// f2 fused plane forward (32 < H, W <= 64); E per orientation as in the staged passes
#ifndef TVP_PLANE_WPB
#define TVP_PLANE_WPB 8
#endif
template <typename T, int ER, int EC, bool LSP>
static cudaError_t plane_fwd_t(const PlaneFwdArgs<T>& a0, cudaStream_t s) {
    constexpr int WPB = TVP_PLANE_WPB;
    PlaneFwdArgs<T> a = a0;
    a.pw = plane_pitch<T>(a.H, a.W, ER, EC);
    const int PW = a.pw;
    const size_t smem = (size_t)3 * a.H * PW * sizeof(T) + (size_t)WPB * 32 * 4 + (size_t)4 * 16 * 32 * 4;
    auto kern = k_plane_fwd<T, ER, EC, WPB, LSP>;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, smem, a.planes, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T, bool LSP>
cudaError_t launch_plane_fwd_ls(const PlaneFwdArgs<T>& a, cudaStream_t s) {
    const int er = pick_geo(a.W).E, ec = pick_geo(a.H).E;
    if (er == 7 && ec == 7) return plane_fwd_t<T, 7, 7, LSP>(a, s);
    if (er == 7) return plane_fwd_t<T, 7, 8, LSP>(a, s);
    if (ec == 7) return plane_fwd_t<T, 8, 7, LSP>(a, s);
    return plane_fwd_t<T, 8, 8, LSP>(a, s);
}

template <typename T, int ER, int EC>
static cudaError_t plane_bwd_t(const PlaneBwdArgs<T>& a0, cudaStream_t s) {
    constexpr int WPB = TVP_PLANE_WPB;
    PlaneBwdArgs<T> a = a0;
    a.pw = plane_pitch<T>(a.H, a.W, ER, EC);
    const int PW = a.pw;
    const size_t smem = (size_t)2 * a.H * PW * sizeof(T);
    auto kern = k_plane_bwd<T, ER, EC, WPB>;
    int grid = 0;
    cudaError_t e = persistent_grid(kern, WPB * 32, smem, a.planes, grid);
    if (e != cudaSuccess) return e;
    kern<<<grid, WPB * 32, smem, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_plane_bwd(const PlaneBwdArgs<T>& a, cudaStream_t s) {
    const int er = pick_geo(a.W).E, ec = pick_geo(a.H).E;
    if (er == 7 && ec == 7) return plane_bwd_t<T, 7, 7>(a, s);
    if (er == 7) return plane_bwd_t<T, 7, 8>(a, s);
    if (ec == 7) return plane_bwd_t<T, 8, 7>(a, s);
    return plane_bwd_t<T, 8, 8>(a, s);
}

// f2 on a thread-block cluster (tv_cluster.cuh): grid = NC x the clusters that fit the
// device at once (cudaOccupancyMaxActiveClusters), each cluster looping over planes.
// The smem opt-in and the cluster occupancy are cached per (device, kernel, smem).
template <typename K>
static cudaError_t cluster_grid(K kern, int threads, size_t smem, int nc, int64_t work, int& grid) {
    static std::mutex mu;
    static std::unordered_map<OccKey, int, OccKeyHash> cache;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int ncl = 0;
    {
        std::lock_guard<std::mutex> g(mu);
        const OccKey key{dev, reinterpret_cast<const void*>(kern), smem};
        auto it = cache.find(key);
        if (it == cache.end()) {
            if (smem > 48 * 1024) {
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (e != cudaSuccess) return e;
            }
            if (nc > 8) {
                e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e != cudaSuccess) return e;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nc, 1, 1);
            cfg.blockDim = dim3(threads, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = nc;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
            if (e != cudaSuccess) return e;
            cache[key] = ncl;
            if (env_int("TVP_CL_VERBOSE", 0))
                fprintf(stderr, "[tvp] cluster kernel: %d clusters of %d CTAs x %d threads, %zu B smem\n", ncl, nc,
                        threads, smem);
        } else {
            ncl = it->second;
        }
    }
    if (ncl < 1) return cudaErrorInvalidConfiguration;
    grid = (int)std::max<int64_t>(1, std::min<int64_t>(work, ncl)) * nc;
    return cudaSuccess;
}

template <typename K, typename A>
static cudaError_t cluster_launch(K kern, const A& a, int grid, int threads, size_t smem, int nc, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(threads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
    count_launch();
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

// Cluster size per line geometry: TVP_CL_NC14 / TVP_CL_NC8 (A/B knobs) pick 4 or 8 CTAs
// for the E = 14 planes (129..224) and 2 or 4 for the E = 8 planes (65..128).
static int cl_nc14() {
    static const int v = env_int("TVP_CL_NC14", 4) == 8 ? 8 : 4;
    return v;
}
static int cl_nc8() {
    static const int v = env_int("TVP_CL_NC8", 2) == 4 ? 4 : 2;
    return v;
}

template <typename T, int E, int NC, int WPB, bool LSP>
static cudaError_t plane_fwd_cl_t(PlaneFwdArgs<T> a, cudaStream_t s) {
    a.coarse = (coarse_knob() && coarse16_knob()) ? 1 : 0;    // as the staged cold passes
    auto kern = k_plane_fwd_cl<T, E, NC, WPB, LSP>;
    const size_t smem = cl_smem_bytes<T>(a.H, a.W, NC, WPB, true);
    int grid = 0;
    cudaError_t e = cluster_grid(kern, WPB * 32, smem, NC, a.planes, grid);
    if (e != cudaSuccess) return e;
    return cluster_launch(kern, a, grid, WPB * 32, smem, NC, s);
}

template <typename T, bool LSP>
cudaError_t launch_plane_fwd_cl_ls(const PlaneFwdArgs<T>& a, cudaStream_t s) {
    if constexpr (sizeof(T) == 4) {
        if (pick_geo(a.H, 4).E == 14)
            return cl_nc14() == 8 ? plane_fwd_cl_t<T, 14, 8, 8, LSP>(a, s) : plane_fwd_cl_t<T, 14, 4, 16, LSP>(a, s);
        return cl_nc8() == 4 ? plane_fwd_cl_t<T, 8, 4, 8, LSP>(a, s) : plane_fwd_cl_t<T, 8, 2, 16, LSP>(a, s);
    }
    return cudaErrorInvalidValue;
}

template <typename T, int E, int NC, int WPB>
static cudaError_t plane_bwd_cl_t(const PlaneBwdArgs<T>& a, cudaStream_t s) {
    auto kern = k_plane_bwd_cl<T, E, NC, WPB>;
    const size_t smem = cl_smem_bytes<T>(a.H, a.W, NC, WPB, false);
    int grid = 0;
    cudaError_t e = cluster_grid(kern, WPB * 32, smem, NC, a.planes, grid);
    if (e != cudaSuccess) return e;
    return cluster_launch(kern, a, grid, WPB * 32, smem, NC, s);
}

template <typename T>
cudaError_t launch_plane_bwd_cl(const PlaneBwdArgs<T>& a, cudaStream_t s) {
    if constexpr (sizeof(T) == 4) {
        if (pick_geo(a.H, 4).E == 14)
            return cl_nc14() == 8 ? plane_bwd_cl_t<T, 14, 8, 8>(a, s) : plane_bwd_cl_t<T, 14, 4, 16>(a, s);
        return cl_nc8() == 4 ? plane_bwd_cl_t<T, 8, 4, 8>(a, s) : plane_bwd_cl_t<T, 8, 2, 16>(a, s);
    }
    return cudaErrorInvalidValue;
}

// f4: a cluster of NCTA = 2..16 CTAs (the smallest power of two that holds the row), each
// CTA 16 warps x 32 lanes x E samples in registers (E = 16 fp32, 8 fp64).
static int long_ncta(int64_t n, int esz) {
    const int64_t per = long_row_per_cta(esz);
    const int64_t c = (n + per - 1) / per;
    return c <= 2 ? 2 : (c <= 4 ? 4 : (c <= 8 ? 8 : 16));   // 16: fp64 only (kMaxLine1DF32 = 8 CTAs)
}
template <typename T, int NCTA, bool PE, bool LSP>
static cudaError_t row_fwd_cl_t(const RowFwdArgs<T>& a, cudaStream_t s) {
    constexpr int E = sizeof(T) == 4 ? 16 : 8, WPL = 16;
    auto kern = k_row_fwd_cl<T, E, WPL, NCTA, PE, LSP>;
    const size_t smem = long_comm_bytes<T>(WPL * NCTA, WPL);
    int grid = 0;
    cudaError_t e = cluster_grid(kern, WPL * 32, smem, NCTA, a.nlines, grid);
    if (e != cudaSuccess) return e;
    return cluster_launch(kern, a, grid, WPL * 32, smem, NCTA, s);
}
template <typename T, bool LSP>
cudaError_t launch_row_fwd_long(const RowFwdArgs<T>& a, bool per_edge, cudaStream_t s) {
    switch (long_ncta(a.n, (int)sizeof(T))) {
        case 2: return per_edge ? row_fwd_cl_t<T, 2, true, LSP>(a, s) : row_fwd_cl_t<T, 2, false, LSP>(a, s);
        case 4: return per_edge ? row_fwd_cl_t<T, 4, true, LSP>(a, s) : row_fwd_cl_t<T, 4, false, LSP>(a, s);
        case 8: return per_edge ? row_fwd_cl_t<T, 8, true, LSP>(a, s) : row_fwd_cl_t<T, 8, false, LSP>(a, s);
        default:
            if constexpr (sizeof(T) == 8)
                return per_edge ? row_fwd_cl_t<T, 16, true, LSP>(a, s) : row_fwd_cl_t<T, 16, false, LSP>(a, s);
            return cudaErrorInvalidValue;           // fp32 rows stop at 8 CTAs (kMaxLine1DF32)
    }
}
template <typename T, int NCTA, bool PE>
static cudaError_t row_bwd_cl_t(const RowBwdArgs<T>& a, cudaStream_t s) {
    constexpr int E = sizeof(T) == 4 ? 16 : 8, WPL = 16;
    auto kern = k_row_bwd_cl<T, E, WPL, NCTA, PE>;
    const size_t smem = long_comm_bytes<T>(WPL * NCTA);
    int grid = 0;
    cudaError_t e = cluster_grid(kern, WPL * 32, smem, NCTA, a.nlines, grid);
    if (e != cudaSuccess) return e;
    return cluster_launch(kern, a, grid, WPL * 32, smem, NCTA, s);
}
template <typename T>
cudaError_t launch_row_bwd_long(const RowBwdArgs<T>& a, bool per_edge, cudaStream_t s) {
    switch (long_ncta(a.n, (int)sizeof(T))) {
        case 2: return per_edge ? row_bwd_cl_t<T, 2, true>(a, s) : row_bwd_cl_t<T, 2, false>(a, s);
        case 4: return per_edge ? row_bwd_cl_t<T, 4, true>(a, s) : row_bwd_cl_t<T, 4, false>(a, s);
        case 8: return per_edge ? row_bwd_cl_t<T, 8, true>(a, s) : row_bwd_cl_t<T, 8, false>(a, s);
        default:
            if constexpr (sizeof(T) == 8) return per_edge ? row_bwd_cl_t<T, 16, true>(a, s) : row_bwd_cl_t<T, 16, false>(a, s);
            return cudaErrorInvalidValue;
    }
}
#define TVP_INST_LONG_FWD(T, LSP) \
    template cudaError_t launch_row_fwd_long<T, LSP>(const RowFwdArgs<T>&, bool, cudaStream_t);
#define TVP_INST_LONG_BWD(T) template cudaError_t launch_row_bwd_long<T>(const RowBwdArgs<T>&, bool, cudaStream_t);

#define TVP_INST_CLUSTER(T)                                                                        \
    template cudaError_t launch_plane_fwd_cl_ls<T, false>(const PlaneFwdArgs<T>&, cudaStream_t);     \
    template cudaError_t launch_plane_fwd_cl_ls<T, true>(const PlaneFwdArgs<T>&, cudaStream_t);      \
    template cudaError_t launch_plane_bwd_cl<T>(const PlaneBwdArgs<T>&, cudaStream_t);

// Explicit instantiations, split over several translation units (tv_inst_*.cu) so the
// build compiles them in parallel.
#define TVP_INST_ROWFWD(T, LSP) template cudaError_t launch_row_fwd_ls<T, LSP>(RowFwdArgs<T>, bool, bool, cudaStream_t);
#define TVP_INST_COLFWD(T, LSP) template cudaError_t launch_col_fwd_ls<T, LSP>(ColFwdArgs<T>, cudaStream_t);
#define TVP_INST_PLANE(T, LSP) template cudaError_t launch_plane_fwd_ls<T, LSP>(const PlaneFwdArgs<T>&, cudaStream_t);
#define TVP_INST_BWD(T)                                                                            \
    template cudaError_t row_fwd_prepass<T>(RowFwdArgs<T>&, bool, bool, cudaStream_t);             \
    template cudaError_t launch_plane_bwd<T>(const PlaneBwdArgs<T>&, cudaStream_t);                \
    template cudaError_t launch_row_bwd<T>(const RowBwdArgs<T>&, bool, bool, cudaStream_t);        \
    template cudaError_t launch_col_bwd<T>(ColBwdArgs<T>, cudaStream_t);                           \
    template cudaError_t launch_lam_reduce<T>(const LamReduceArgs<T>&, cudaStream_t);              \
    template cudaError_t launch_softplus<T>(const T*, T*, const T*, T*, int64_t, bool, cudaStream_t);\
    template cudaError_t launch_axpby<T>(const T*, T*, T, T, int64_t, cudaStream_t);

}  // namespace tvp
