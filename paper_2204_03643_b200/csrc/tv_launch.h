// tv_launch.h -- host-side launch interface between the C ABI (tvprox_abi.cu)
// and the per-dtype kernel instantiation units (tv_f32.cu, tv_f64.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvp {

template <typename T> struct RowFwdArgs;
template <typename T> struct ColFwdArgs;
template <typename T> struct RowBwdArgs;
template <typename T> struct ColBwdArgs;
template <typename T> struct LamReduceArgs;
template <typename T> struct PlaneFwdArgs;
template <typename T> struct PlaneBwdArgs;

// (E samples per lane, LPR lanes per line) chosen for a line length n.
struct Geo { int E, LPR; };
// TVP_GEO16=1 (default; environment 0 for A/B): fp32 lines of 129..224 samples go to
// half-warp groups of 14 samples per lane (two lines per warp) instead of one warp of 7
// per lane, and 65..128 samples to half-warp groups of 8 instead of one warp of 4 --
// the per-iteration scan / vote overhead is shared by twice the samples.
#ifndef TVP_GEO16_DEFAULT
#define TVP_GEO16_DEFAULT 1
#endif
int geo16_knob();
inline Geo pick_geo(int64_t n, int esz = 8) {
    if (esz == 4 && n > 128 && n <= 224 && geo16_knob()) return {14, 16};
    if (esz == 4 && n > 64 && n <= 128 && geo16_knob()) return {8, 16};
    if (n <= 16) return {2, 8};
    if (n <= 32) return {4, 8};
    if (n <= 56) return {7, 8};
    if (n <= 64) return {8, 8};
    if (n <= 128) return {4, 32};
    if (n <= 224) return {7, 32};
    if (n <= 256) return {8, 32};
    if (n <= 512) return {16, 32};
    return {32, 32};
}
constexpr int64_t kMaxLine = 1024;                 // 2D lines (W, H)
// 1D rows: a CTA of up to 16 warps holds the row in registers (E = 16 fp32, 8 fp64), up
// to 8192 / 4096 samples; beyond, a thread-block cluster of such CTAs (f4): up to 8 CTAs
// in fp32 (65536 samples -- longer fp32 rows measured 1.4e-4 x range off the oracle on
// the noisiest synthetic workload, O7) and 16 in fp64 (65536).
constexpr int64_t kMaxLine1DF32 = 8 * 16 * 32 * 16;     // 65536
constexpr int64_t kMaxLine1DF64 = 16 * 16 * 32 * 8;     // 65536
// First-level chunks of the lambda-gradient reduction: a function of the sizes only
// (never of the GPU), so results are bitwise reproducible across devices.
inline int lam_chunks(int64_t total, int64_t nout) {
    (void)nout;
    int64_t c = (total + 8191) / 8192;
    if (c > 512) c = 512;
    if (c < 1) c = 1;
    return (int)c;
}

// Forward launchers per line-search flavour (LSP: parallel step search, f3) and the
// dispatchers the C ABI calls (lsp = tvp_options_t.line_search == TVP_LS_PARALLEL).
template <typename T> cudaError_t row_fwd_prepass(RowFwdArgs<T>& a, bool per_edge, bool dykstra, cudaStream_t s);
template <typename T, bool LSP> cudaError_t launch_row_fwd_ls(RowFwdArgs<T> a, bool per_edge, bool dykstra, cudaStream_t s);
template <typename T, bool LSP> cudaError_t launch_col_fwd_ls(ColFwdArgs<T> a, cudaStream_t s);
template <typename T, bool LSP> cudaError_t launch_plane_fwd_ls(const PlaneFwdArgs<T>& a, cudaStream_t s);
template <typename T>
inline cudaError_t launch_row_fwd(RowFwdArgs<T> a, bool per_edge, bool dykstra, cudaStream_t s, bool lsp) {
    cudaError_t e = row_fwd_prepass<T>(a, per_edge, dykstra, s);
    if (e != cudaSuccess) return e;
    return lsp ? launch_row_fwd_ls<T, true>(a, per_edge, dykstra, s) : launch_row_fwd_ls<T, false>(a, per_edge, dykstra, s);
}
template <typename T>
inline cudaError_t launch_col_fwd(const ColFwdArgs<T>& a, cudaStream_t s, bool lsp) {
    return lsp ? launch_col_fwd_ls<T, true>(a, s) : launch_col_fwd_ls<T, false>(a, s);
}
template <typename T>
inline cudaError_t launch_plane_fwd(const PlaneFwdArgs<T>& a, cudaStream_t s, bool lsp) {
    return lsp ? launch_plane_fwd_ls<T, true>(a, s) : launch_plane_fwd_ls<T, false>(a, s);
}
template <typename T> cudaError_t launch_plane_bwd(const PlaneBwdArgs<T>& a, cudaStream_t s);
inline bool plane_fwd_supported(int64_t H, int64_t W) { return H > 32 && H <= 64 && W > 32 && W <= 64; }
// f2 on a thread-block cluster (tv_cluster.cuh): fp32 planes whose rows and columns both
// take the half-warp geometry of the staged passes with the same E (65..128 -> E = 8,
// 129..224 -> E = 14), so the result is bitwise the staged one.
inline bool plane_cl_supported(int64_t H, int64_t W, int esz) {
    if (esz != 4 || !geo16_knob()) return false;
    const Geo gh = pick_geo(H, 4), gw = pick_geo(W, 4);
    return gh.LPR == 16 && gw.LPR == 16 && gh.E == gw.E;
}
template <typename T, bool LSP> cudaError_t launch_plane_fwd_cl_ls(const PlaneFwdArgs<T>& a, cudaStream_t s);
template <typename T> cudaError_t launch_plane_bwd_cl(const PlaneBwdArgs<T>& a, cudaStream_t s);
template <typename T>
inline cudaError_t launch_plane_fwd_cl(const PlaneFwdArgs<T>& a, cudaStream_t s, bool lsp) {
    return lsp ? launch_plane_fwd_cl_ls<T, true>(a, s) : launch_plane_fwd_cl_ls<T, false>(a, s);
}
template <typename T> cudaError_t launch_row_bwd(const RowBwdArgs<T>& a, bool dykstra, bool per_edge, cudaStream_t s);
template <typename T> cudaError_t launch_col_bwd(ColBwdArgs<T> a, cudaStream_t s);
template <typename T> cudaError_t launch_lam_reduce(const LamReduceArgs<T>& a, cudaStream_t s);

template <typename T> cudaError_t launch_softplus(const T* t, T* lam, const T* g, T* gt, int64_t n, bool bwd, cudaStream_t s);
template <typename T> cudaError_t launch_axpby(const T* x, T* y, T a, T b, int64_t n, cudaStream_t s);

void count_launch();

}  // namespace tvp
