// tvprox_abi.cu -- the extern "C" boundary of libtvprox.so (include/tvprox.h):
// argument validation, workspace carving, the Dykstra pass schedule of
// Algorithm 1 and its reverse, and dispatch to the
// per-dtype launchers.  No compute happens here; every step runs in kernels.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/tvprox.h"
#include "tv_kernels.cuh"
#include "tv_launch.h"

namespace tvp {
static thread_local std::string g_err;
static thread_local int64_t g_launches = 0;
void count_launch() { ++g_launches; }
// f2 fused on-chip 2D path: the calling thread's default for tvp_options_t.fused2d = -1
// (initially on; TVP_FUSED2D=0 in the environment -> staged).
static bool fused2d_env() {
    static const bool v = [] {
        const char* e = getenv("TVP_FUSED2D");
        return !(e && atoi(e) == 0);
    }();
    return v;
}
// TVP_FUSED2D=2: the default also takes the thread-block-cluster planes (65..224 per side),
// which are otherwise only used on explicit request (tvp_options_t.fused2d = 1): on B200
// they measure slower than the staged passes for C5.
static bool cluster_env() {
    static const bool v = [] {
        const char* e = getenv("TVP_FUSED2D");
        return e && atoi(e) == 2;
    }();
    return v;
}
static thread_local int g_fused2d = -1;     // -1: not set on this thread (environment default)
int geo16_knob() {
    static const int v = [] {
        const char* e = getenv("TVP_GEO16");
        return e ? atoi(e) : TVP_GEO16_DEFAULT;
    }();
    return v;
}
}  // namespace tvp

using namespace tvp;

static tvp_status_t fail(tvp_status_t st, const char* msg) {
    g_err = msg;
    return st;
}
static tvp_status_t cuda_status(cudaError_t e, const char* where) {
    if (e == cudaSuccess) return TVP_OK;
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return TVP_ECUDA;
}
static size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Resolved per-call options (tvp_options_t, include/tvprox.h).
struct Opts {
    bool fused2d;
    bool cluster;       // f2 also for the thread-block-cluster planes
    bool lsp;
    int ls_after;
    int32_t* diag;
    int32_t* hist;
};
static bool resolve_opts(const tvp_options_t* o, Opts& r) {
    const int f = o ? o->fused2d : -1;
    const int ls = o ? o->line_search : TVP_LS_BACKTRACK;
    const int after = o ? o->ls_after : 0;
    if (f < -1 || f > 1 || (ls != TVP_LS_BACKTRACK && ls != TVP_LS_PARALLEL) || after < 0) return false;
    r.fused2d = f == -1 ? (g_fused2d == -1 ? fused2d_env() : g_fused2d != 0) : f != 0;
    r.cluster = f == 1 || (f == -1 && g_fused2d == -1 && cluster_env());
    r.lsp = ls == TVP_LS_PARALLEL;
    r.ls_after = after == 0 ? kLsAfterDefault : after;
    r.diag = o ? o->diag : nullptr;
    r.hist = o ? o->iter_hist : nullptr;
    return true;
}
static int64_t mask_words(int64_t n) { return n <= 1 ? 0 : (n - 1 + 15) / 16; }

extern "C" {

int tvp_version(void) { return 100; }
const char* tvp_last_error(void) { return g_err.c_str(); }
int64_t tvp_launch_count(int reset) {
    int64_t v = g_launches;
    if (reset) g_launches = 0;
    return v;
}
const char* tvp_status_string(tvp_status_t s) {
    switch (s) {
        case TVP_OK: return "TVP_OK";
        case TVP_EINVAL: return "TVP_EINVAL: invalid argument";
        case TVP_EUNSUPPORTED: return "TVP_EUNSUPPORTED: unsupported size or mode";
        case TVP_ECUDA: return "TVP_ECUDA: CUDA launch or driver error";
        default: return "TVP_UNKNOWN";
    }
}
int64_t tvp_max_line(tvp_dtype_t dt) { (void)dt; return kMaxLine; }
int tvp_set_fused2d(int enable) {
    const int prev = g_fused2d == -1 ? (fused2d_env() ? 1 : 0) : g_fused2d;
    g_fused2d = enable != 0 ? 1 : 0;
    return prev;
}
void tvp_options_default(tvp_options_t* o) {
    if (!o) return;
    o->fused2d = -1;
    o->line_search = TVP_LS_BACKTRACK;
    o->ls_after = 0;
    o->diag = nullptr;
    o->iter_hist = nullptr;
}
int64_t tvp_max_line_1d(tvp_dtype_t dt) { return dt == TVP_F64 ? kMaxLine1DF64 : kMaxLine1DF32; }
size_t tv1d_mask_words(int64_t n) { return (size_t)mask_words(n); }

size_t tv1d_bwd_workspace_bytes(tvp_dtype_t dt, int64_t batch, tvp_lam_mode_t lm) {
    if (lm != TVP_LAM_SCALAR || batch <= 0) return 0;
    const size_t esz = dt == TVP_F64 ? 8 : 4;
    return align256((size_t)batch * esz) + align256(512 * esz);
}

size_t tv2d_saved_bytes(int64_t N, int64_t C, int64_t H, int64_t W, int iters) {
    if (N < 0 || C < 0 || H < 1 || W < 1 || iters < 1) return 0;
    const int64_t planes = N * C;
    return (size_t)iters * planes * (H * mask_words(W) + W * mask_words(H)) * 4;
}

struct Ws2D {
    size_t z, p, q, rmask, cmask, lam, lam2, total;
};
static Ws2D ws_layout(size_t esz, int64_t N, int64_t C, int64_t H, int64_t W, int iters) {
    const int64_t planes = N * C;
    const size_t plane_b = align256((size_t)planes * H * W * esz);
    Ws2D w{};
    size_t off = 0;
    w.z = off; off += plane_b;
    w.p = off; off += plane_b;
    w.q = off; off += plane_b;
    w.rmask = off; off += align256((size_t)planes * H * mask_words(W) * 4);
    w.cmask = off; off += align256((size_t)planes * W * mask_words(H) * 4);
    w.lam = off; off += align256((size_t)planes * iters * (H + W) * esz);
    w.lam2 = off; off += align256((size_t)512 * (planes > 0 ? planes : 1) * esz);
    w.total = off;
    return w;
}

size_t tv2d_workspace_bytes(tvp_dtype_t dt, int64_t N, int64_t C, int64_t H, int64_t W, int iters) {
    if (N < 0 || C < 0 || H < 1 || W < 1 || iters < 1) return 0;
    return ws_layout(dt == TVP_F64 ? 8 : 4, N, C, H, W, iters).total;
}

}  // extern "C"

// ------------------------------------------------------------------------ 1D
template <typename T>
static tvp_status_t tv1d_fwd_impl(const void* y, void* x, int64_t batch, int64_t n, int64_t stride,
                                  const void* lam, tvp_lam_mode_t lm, double lam_scalar, uint32_t* mask,
                                  int32_t* row_iters, cudaStream_t s, const uint32_t* mask_in, const Opts& o) {
    RowFwdArgs<T> a{};
    a.src0 = static_cast<const T*>(y);
    a.src1 = nullptr;
    a.dst0 = static_cast<T*>(x);
    a.dst1 = nullptr;
    a.lam = static_cast<const T*>(lam);
    a.lam_mode = (int)lm;
    a.lam_scalar = (T)lam_scalar;
    a.nlines = batch;
    a.n = (int)n;
    a.stride = stride;
    a.lines_per_plane = 1;
    a.C = 1;
    a.mask_in = mask_in;
    a.mask_out = mask;
    a.mw = (int)mask_words(n);
    a.row_iters = row_iters;
    a.iters_max = nullptr;
    a.ls_after = o.ls_after;
    a.diag = o.diag;
    a.hist = o.hist;
    return cuda_status(launch_row_fwd<T>(a, lm == TVP_LAM_PER_EDGE, false, s, o.lsp), "tv1d_prox_fwd");
}

extern "C" tvp_status_t tv1d_prox_fwd_ex(tvp_dtype_t dt, const void* y, void* x, int64_t batch, int64_t n,
                                         int64_t stride, const void* lam, tvp_lam_mode_t lm, double lam_scalar,
                                         const uint32_t* mask_in, uint32_t* mask_out, int32_t* row_iters,
                                         const tvp_options_t* opts, tvp_stream_t stream) {
    Opts o;
    if (!resolve_opts(opts, o)) return fail(TVP_EINVAL, "tv1d_prox_fwd: invalid tvp_options_t");
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv1d_prox_fwd: bad dtype");
    if (batch < 0 || n < 1 || stride < n) return fail(TVP_EINVAL, "tv1d_prox_fwd: need batch >= 0, n >= 1, stride >= n");
    if (lm != TVP_LAM_SCALAR && lm != TVP_LAM_PER_ROW && lm != TVP_LAM_PER_EDGE)
        return fail(TVP_EINVAL, "tv1d_prox_fwd: lam mode must be SCALAR, PER_ROW or PER_EDGE");
    if (lm == TVP_LAM_SCALAR && !(std::isfinite(lam_scalar) && lam_scalar >= 0.0))
        return fail(TVP_EINVAL, "tv1d_prox_fwd: lam_scalar must be finite and >= 0");
    if (batch == 0) return TVP_OK;
    if (!y || !x) return fail(TVP_EINVAL, "tv1d_prox_fwd: NULL y or x");
    if (lm != TVP_LAM_SCALAR && !lam) return fail(TVP_EINVAL, "tv1d_prox_fwd: NULL lam");
    if (n > tvp_max_line_1d(dt)) return fail(TVP_EUNSUPPORTED, "tv1d_prox_fwd: n > tvp_max_line_1d()");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dt == TVP_F32
               ? tv1d_fwd_impl<float>(y, x, batch, n, stride, lam, lm, lam_scalar, mask_out, row_iters, s, mask_in, o)
               : tv1d_fwd_impl<double>(y, x, batch, n, stride, lam, lm, lam_scalar, mask_out, row_iters, s, mask_in, o);
}

extern "C" tvp_status_t tv1d_prox_fwd(tvp_dtype_t dt, const void* y, void* x, int64_t batch, int64_t n,
                                      int64_t stride, const void* lam, tvp_lam_mode_t lm, double lam_scalar,
                                      uint32_t* mask, int32_t* row_iters, tvp_stream_t stream) {
    return tv1d_prox_fwd_ex(dt, y, x, batch, n, stride, lam, lm, lam_scalar, nullptr, mask, row_iters, nullptr,
                            stream);
}

extern "C" tvp_status_t tv1d_prox_fwd_warm(tvp_dtype_t dt, const void* y, void* x, int64_t batch, int64_t n,
                                           int64_t stride, const void* lam, tvp_lam_mode_t lm, double lam_scalar,
                                           const uint32_t* mask_in, uint32_t* mask_out, int32_t* row_iters,
                                           tvp_stream_t stream) {
    if (n > 1 && batch > 0 && !mask_in) return fail(TVP_EINVAL, "tv1d_prox_fwd_warm: NULL mask_in");
    return tv1d_prox_fwd_ex(dt, y, x, batch, n, stride, lam, lm, lam_scalar, mask_in, mask_out, row_iters, nullptr,
                            stream);
}

template <typename T>
static tvp_status_t tv1d_bwd_impl(const void* gx, const uint32_t* mask, void* gy, void* glam, int64_t batch,
                                  int64_t n, int64_t stride, tvp_lam_mode_t lm, void* ws, cudaStream_t s) {
    RowBwdArgs<T> a{};
    a.A = static_cast<const T*>(gx);
    a.B = nullptr;
    a.out = static_cast<T*>(gy);
    a.mask = mask;
    a.mw = (int)mask_words(n);
    a.nlines = batch;
    a.n = (int)n;
    a.stride = stride;
    a.lam_lpp = 1;
    a.lam_pstride = 1;
    a.lam_line = nullptr;
    a.lam_edge = nullptr;
    if (glam) {
        if (lm == TVP_LAM_PER_ROW) a.lam_line = static_cast<T*>(glam);
        else if (lm == TVP_LAM_SCALAR) a.lam_line = static_cast<T*>(ws);
        else a.lam_edge = static_cast<T*>(glam);
    }
    cudaError_t e = launch_row_bwd<T>(a, false, lm == TVP_LAM_PER_EDGE && glam, s);
    if (e != cudaSuccess) return cuda_status(e, "tv1d_prox_bwd");
    if (glam && lm == TVP_LAM_SCALAR) {
        LamReduceArgs<T> r{};
        r.part = static_cast<const T*>(ws);
        r.out = static_cast<T*>(glam);
        r.nout = 1;
        r.reps = 1;
        r.rep_stride = 0;
        r.q_stride = 0;
        r.seglen = batch;
        r.nchunk = lam_chunks(batch, 1);
        r.scratch = reinterpret_cast<T*>(static_cast<char*>(ws) + align256((size_t)batch * sizeof(T)));
        e = launch_lam_reduce<T>(r, s);
    }
    return cuda_status(e, "tv1d_prox_bwd");
}

extern "C" tvp_status_t tv1d_prox_bwd(tvp_dtype_t dt, const void* grad_x, const uint32_t* mask, void* grad_y,
                                      void* grad_lam, int64_t batch, int64_t n, int64_t stride,
                                      tvp_lam_mode_t lm, void* workspace, tvp_stream_t stream) {
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv1d_prox_bwd: bad dtype");
    if (batch < 0 || n < 1 || stride < n) return fail(TVP_EINVAL, "tv1d_prox_bwd: need batch >= 0, n >= 1, stride >= n");
    if (lm != TVP_LAM_SCALAR && lm != TVP_LAM_PER_ROW && lm != TVP_LAM_PER_EDGE)
        return fail(TVP_EINVAL, "tv1d_prox_bwd: lam mode must be SCALAR, PER_ROW or PER_EDGE");
    if (batch == 0) {
        if (grad_lam && lm == TVP_LAM_SCALAR) {
            cudaError_t e = cudaMemsetAsync(grad_lam, 0, dt == TVP_F64 ? 8 : 4, reinterpret_cast<cudaStream_t>(stream));
            return cuda_status(e, "tv1d_prox_bwd");
        }
        return TVP_OK;
    }
    if (!grad_x || !grad_y) return fail(TVP_EINVAL, "tv1d_prox_bwd: NULL grad_x or grad_y");
    if (n > 1 && !mask) return fail(TVP_EINVAL, "tv1d_prox_bwd: NULL mask");
    if (grad_lam && lm == TVP_LAM_SCALAR && !workspace) return fail(TVP_EINVAL, "tv1d_prox_bwd: NULL workspace");
    if (n > tvp_max_line_1d(dt)) return fail(TVP_EUNSUPPORTED, "tv1d_prox_bwd: n > tvp_max_line_1d()");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dt == TVP_F32 ? tv1d_bwd_impl<float>(grad_x, mask, grad_y, grad_lam, batch, n, stride, lm, workspace, s)
                         : tv1d_bwd_impl<double>(grad_x, mask, grad_y, grad_lam, batch, n, stride, lm, workspace, s);
}

// ------------------------------------------------------------------------ 2D
static bool lam2d_ok(tvp_lam_mode_t lm, const void* lam, double lam_scalar) {
    if (lm == TVP_LAM_SCALAR) return std::isfinite(lam_scalar) && lam_scalar >= 0.0;
    if (lm == TVP_LAM_PER_CHANNEL || lm == TVP_LAM_PER_PLANE) return lam != nullptr;
    return false;
}

template <typename T>
static tvp_status_t tv2d_fwd_impl(const void* Xv, void* Yv, int64_t N, int64_t C, int64_t H, int64_t W,
                                  const void* lam, tvp_lam_mode_t lm, double lam_scalar, int K, void* saved,
                                  void* workspace, int32_t* line_iters, cudaStream_t s, const Opts& o) {
    const int64_t planes = N * C;
    const Ws2D L = ws_layout(sizeof(T), N, C, H, W, K);
    char* ws = static_cast<char*>(workspace);
    T* Z = reinterpret_cast<T*>(ws + L.z);
    T* P = reinterpret_cast<T*>(ws + L.p);
    T* Q = reinterpret_cast<T*>(ws + L.q);
    const int64_t mwr = mask_words(W), mwc = mask_words(H);
    const int64_t rset = planes * H * mwr, cset = planes * W * mwc;
    uint32_t* sv = static_cast<uint32_t*>(saved);
    uint32_t* rws = reinterpret_cast<uint32_t*>(ws + L.rmask);
    uint32_t* cws = reinterpret_cast<uint32_t*>(ws + L.cmask);
    const T* X = static_cast<const T*>(Xv);
    T* Y = static_cast<T*>(Yv);
    if (line_iters) {
        cudaError_t e = cudaMemsetAsync(line_iters, 0, sizeof(int32_t) * 2 * K, s);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_fwd");
    }
    const bool cl = o.cluster && plane_cl_supported(H, W, (int)sizeof(T));
    if ((o.fused2d && plane_fwd_supported(H, W)) || cl) {
        // f2: the whole plane stays on chip for all K passes (no Z/P/Q workspace traffic):
        // one CTA per plane up to 64 x 64, a thread-block cluster up to 224 x 224
        PlaneFwdArgs<T> f{};
        f.X = X;
        f.Y = Y;
        f.lam = static_cast<const T*>(lam);
        f.lam_mode = (int)lm;
        f.lam_scalar = (T)lam_scalar;
        f.C = (int)(C > 0 ? C : 1);
        f.planes = planes;
        f.H = (int)H;
        f.W = (int)W;
        f.K = K;
        f.saved = sv;
        f.mwr = (int)mwr;
        f.mwc = (int)mwc;
        f.iters_max = line_iters;
        f.ls_after = o.ls_after;
        f.diag = o.diag;
        f.hist = o.hist;
        if (cl) return cuda_status(launch_plane_fwd_cl<T>(f, s, o.lsp), "tv2d_prox_fwd(fused cluster)");
        return cuda_status(launch_plane_fwd<T>(f, s, o.lsp), "tv2d_prox_fwd(fused)");
    }
    for (int k = 1; k <= K; ++k) {
        // ---- row pass (Alg. 1 lines 3-6): Z = rowprox(Y + P); P <- (Y + P) - Z
        RowFwdArgs<T> r{};
        r.src0 = (k == 1) ? X : Y;
        r.src1 = (k == 1) ? nullptr : P;
        r.dst0 = Z;
        r.dst1 = P;
        r.lam = static_cast<const T*>(lam);
        r.lam_mode = (int)lm;
        r.lam_scalar = (T)lam_scalar;
        r.nlines = planes * H;
        r.n = (int)W;
        r.stride = W;
        r.lines_per_plane = H;
        r.C = (int)(C > 0 ? C : 1);
        r.mw = (int)mwr;
        r.mask_out = sv ? sv + (k - 1) * rset : rws;
        r.mask_in = (k == 1) ? nullptr : (sv ? sv + (k - 2) * rset : rws);
        r.row_iters = nullptr;
        r.iters_max = line_iters ? line_iters + 2 * (k - 1) : nullptr;
        r.ls_after = o.ls_after;
        r.diag = o.diag;
        r.hist = o.hist ? o.hist + (int64_t)(2 * (k - 1)) * TVP_HIST_BINS : nullptr;
        cudaError_t e = launch_row_fwd<T>(r, false, true, s, o.lsp);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_fwd(row)");
        // ---- column pass (lines 7-10): Y = colprox(Z + Q); Q <- (Z + Q) - Y
        ColFwdArgs<T> c{};
        c.Z = Z;
        c.Q = (k == 1) ? nullptr : Q;
        c.Y = Y;
        c.Qout = (k == K) ? nullptr : Q;
        c.lam = static_cast<const T*>(lam);
        c.lam_mode = (int)lm;
        c.lam_scalar = (T)lam_scalar;
        c.C = (int)(C > 0 ? C : 1);
        c.planes = planes;
        c.H = (int)H;
        c.W = (int)W;
        c.mw = (int)mwc;
        uint32_t* cbase = sv ? sv + (int64_t)K * rset : nullptr;
        c.mask_out = sv ? cbase + (k - 1) * cset : cws;
        c.mask_in = (k == 1) ? nullptr : (sv ? cbase + (k - 2) * cset : cws);
        c.iters_max = line_iters ? line_iters + 2 * (k - 1) + 1 : nullptr;
        c.ls_after = o.ls_after;
        c.diag = o.diag;
        c.hist = o.hist ? o.hist + (int64_t)(2 * (k - 1) + 1) * TVP_HIST_BINS : nullptr;
        e = launch_col_fwd<T>(c, s, o.lsp);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_fwd(col)");
    }
    return TVP_OK;
}

extern "C" tvp_status_t tv2d_prox_fwd_ex(tvp_dtype_t dt, const void* X, void* Y, int64_t N, int64_t C, int64_t H,
                                         int64_t W, const void* lam, tvp_lam_mode_t lm, double lam_scalar, int iters,
                                         void* saved, void* workspace, int32_t* line_iters,
                                         const tvp_options_t* opts, tvp_stream_t stream) {
    Opts o;
    if (!resolve_opts(opts, o)) return fail(TVP_EINVAL, "tv2d_prox_fwd: invalid tvp_options_t");
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv2d_prox_fwd: bad dtype");
    if (N < 0 || C < 0 || H < 1 || W < 1 || iters < 1)
        return fail(TVP_EINVAL, "tv2d_prox_fwd: need N, C >= 0, H, W >= 1, iters >= 1");
    if (!lam2d_ok(lm, lam, lam_scalar)) return fail(TVP_EINVAL, "tv2d_prox_fwd: invalid lam / lam mode");
    if (N * C == 0) return TVP_OK;
    if (!X || !Y || !workspace) return fail(TVP_EINVAL, "tv2d_prox_fwd: NULL X, Y or workspace");
    if (H > kMaxLine || W > kMaxLine) return fail(TVP_EUNSUPPORTED, "tv2d_prox_fwd: H or W > tvp_max_line()");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dt == TVP_F32
               ? tv2d_fwd_impl<float>(X, Y, N, C, H, W, lam, lm, lam_scalar, iters, saved, workspace, line_iters, s, o)
               : tv2d_fwd_impl<double>(X, Y, N, C, H, W, lam, lm, lam_scalar, iters, saved, workspace, line_iters, s, o);
}

extern "C" tvp_status_t tv2d_prox_fwd(tvp_dtype_t dt, const void* X, void* Y, int64_t N, int64_t C, int64_t H,
                                      int64_t W, const void* lam, tvp_lam_mode_t lm, double lam_scalar, int iters,
                                      void* saved, void* workspace, int32_t* line_iters, tvp_stream_t stream) {
    return tv2d_prox_fwd_ex(dt, X, Y, N, C, H, W, lam, lm, lam_scalar, iters, saved, workspace, line_iters, nullptr,
                            stream);
}

template <typename T>
static tvp_status_t tv2d_bwd_impl(const void* GYv, const void* saved, void* GXv, void* glam, int64_t N, int64_t C,
                                  int64_t H, int64_t W, tvp_lam_mode_t lm, int K, void* workspace, cudaStream_t s,
                                  const Opts& o) {
    const int64_t planes = N * C;
    const Ws2D L = ws_layout(sizeof(T), N, C, H, W, K);
    char* ws = static_cast<char*>(workspace);
    T* B = reinterpret_cast<T*>(ws + L.z);
    T* lampart = reinterpret_cast<T*>(ws + L.lam);
    const int64_t mwr = mask_words(W), mwc = mask_words(H);
    const int64_t rset = planes * H * mwr, cset = planes * W * mwc;
    const uint32_t* sv = static_cast<const uint32_t*>(saved);
    const T* G = static_cast<const T*>(GYv);
    T* GX = static_cast<T*>(GXv);
    const int64_t HW2 = H + W;
    const bool cl = o.cluster && plane_cl_supported(H, W, (int)sizeof(T));
    const bool fused = (o.fused2d && plane_fwd_supported(H, W)) || cl;
    if (fused) {
        // f2: both adjoint planes stay on chip through all 2K adjoint passes
        PlaneBwdArgs<T> f{};
        f.G = G;
        f.GX = GX;
        f.saved = sv;
        f.planes = planes;
        f.H = (int)H;
        f.W = (int)W;
        f.K = K;
        f.mwr = (int)mwr;
        f.mwc = (int)mwc;
        f.lampart = glam ? lampart : nullptr;
        cudaError_t e = cl ? launch_plane_bwd_cl<T>(f, s) : launch_plane_bwd<T>(f, s);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_bwd(fused)");
    }
    for (int k = K; k >= 1 && !fused; --k) {
        // ---- column adjoint: r = A - B; B <- B + colsegmean_k(r)   (A = G at k = K, B = 0)
        ColBwdArgs<T> c{};
        c.A = (k == K) ? G : GX;
        c.B = (k == K) ? nullptr : B;
        c.Bout = B;
        c.mask = sv + (int64_t)K * rset + (k - 1) * cset;
        c.mw = (int)mwc;
        c.planes = planes;
        c.H = (int)H;
        c.W = (int)W;
        c.lam_line = glam ? lampart + (k - 1) * HW2 + H : nullptr;
        c.lam_pstride = (int64_t)K * HW2;
        cudaError_t e = launch_col_bwd<T>(c, s);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_bwd(col)");
        // ---- row adjoint: r = B - Pbar; A <- Pbar + rowsegmean_k(r)   (Pbar = A, or 0 at k = K)
        RowBwdArgs<T> r{};
        r.A = (k == K) ? nullptr : GX;
        r.B = B;
        r.out = GX;
        r.mask = sv + (k - 1) * rset;
        r.mw = (int)mwr;
        r.nlines = planes * H;
        r.n = (int)W;
        r.stride = W;
        r.lam_line = glam ? lampart + (k - 1) * HW2 : nullptr;
        r.lam_lpp = H;
        r.lam_pstride = (int64_t)K * HW2;
        r.lam_edge = nullptr;
        e = launch_row_bwd<T>(r, true, false, s);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_bwd(row)");
    }
    if (glam) {
        LamReduceArgs<T> q{};
        q.part = lampart;
        q.out = static_cast<T*>(glam);
        const int64_t per_plane = (int64_t)K * HW2;
        if (lm == TVP_LAM_SCALAR) {
            q.nout = 1; q.reps = 1; q.rep_stride = 0; q.q_stride = 0; q.seglen = planes * per_plane;
        } else if (lm == TVP_LAM_PER_CHANNEL) {
            q.nout = C; q.reps = N; q.rep_stride = C * per_plane; q.q_stride = per_plane; q.seglen = per_plane;
        } else {
            q.nout = planes; q.reps = 1; q.rep_stride = 0; q.q_stride = per_plane; q.seglen = per_plane;
        }
        q.nchunk = lam_chunks(q.reps * q.seglen, q.nout);
        q.scratch = reinterpret_cast<T*>(ws + L.lam2);
        cudaError_t e = launch_lam_reduce<T>(q, s);
        if (e != cudaSuccess) return cuda_status(e, "tv2d_prox_bwd(lam)");
    }
    return TVP_OK;
}

extern "C" tvp_status_t tv2d_prox_bwd_ex(tvp_dtype_t dt, const void* grad_Y, const void* saved, void* grad_X,
                                         void* grad_lam, int64_t N, int64_t C, int64_t H, int64_t W,
                                         tvp_lam_mode_t lm, int iters, void* workspace, const tvp_options_t* opts,
                                         tvp_stream_t stream) {
    Opts o;
    if (!resolve_opts(opts, o)) return fail(TVP_EINVAL, "tv2d_prox_bwd: invalid tvp_options_t");
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv2d_prox_bwd: bad dtype");
    if (N < 0 || C < 0 || H < 1 || W < 1 || iters < 1)
        return fail(TVP_EINVAL, "tv2d_prox_bwd: need N, C >= 0, H, W >= 1, iters >= 1");
    if (lm != TVP_LAM_SCALAR && lm != TVP_LAM_PER_CHANNEL && lm != TVP_LAM_PER_PLANE)
        return fail(TVP_EINVAL, "tv2d_prox_bwd: lam mode must be SCALAR, PER_CHANNEL or PER_PLANE");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (N * C == 0) {
        if (grad_lam) {
            size_t cnt = lm == TVP_LAM_SCALAR ? 1 : (lm == TVP_LAM_PER_CHANNEL ? (size_t)C : 0);
            if (cnt) return cuda_status(cudaMemsetAsync(grad_lam, 0, cnt * (dt == TVP_F64 ? 8 : 4), s), "tv2d_prox_bwd");
        }
        return TVP_OK;
    }
    if (!grad_Y || !grad_X || !workspace || !saved) return fail(TVP_EINVAL, "tv2d_prox_bwd: NULL grad_Y, grad_X, saved or workspace");
    if (H > kMaxLine || W > kMaxLine) return fail(TVP_EUNSUPPORTED, "tv2d_prox_bwd: H or W > tvp_max_line()");
    return dt == TVP_F32 ? tv2d_bwd_impl<float>(grad_Y, saved, grad_X, grad_lam, N, C, H, W, lm, iters, workspace, s, o)
                         : tv2d_bwd_impl<double>(grad_Y, saved, grad_X, grad_lam, N, C, H, W, lm, iters, workspace, s, o);
}

extern "C" tvp_status_t tv2d_prox_bwd(tvp_dtype_t dt, const void* grad_Y, const void* saved, void* grad_X,
                                      void* grad_lam, int64_t N, int64_t C, int64_t H, int64_t W,
                                      tvp_lam_mode_t lm, int iters, void* workspace, tvp_stream_t stream) {
    return tv2d_prox_bwd_ex(dt, grad_Y, saved, grad_X, grad_lam, N, C, H, W, lm, iters, workspace, nullptr, stream);
}

// ------------------------------------------------------------ TV layer (f1)
static bool lines_args_ok(int64_t N, int64_t C, int64_t H, int64_t W, int axis) {
    return N >= 0 && C >= 0 && H >= 1 && W >= 1 && (axis == 0 || axis == 1);
}

extern "C" size_t tv2d_lines_workspace_bytes(tvp_dtype_t dt, int64_t N, int64_t C, int64_t H, int64_t W, int axis) {
    if (!lines_args_ok(N, C, H, W, axis)) return 0;
    const size_t esz = dt == TVP_F64 ? 8 : 4;
    const int64_t planes = N * C;
    const int64_t lines = planes * (axis == 0 ? H : W);
    return align256((size_t)lines * esz) + align256((size_t)512 * (planes > 0 ? planes : 1) * esz);
}

template <typename T>
static tvp_status_t lines_fwd_impl(const void* X, void* Y, int64_t N, int64_t C, int64_t H, int64_t W,
                                   const void* lam, tvp_lam_mode_t lm, double lam_scalar, int axis, uint32_t* mask,
                                   cudaStream_t s) {
    const int64_t planes = N * C;
    if (axis == 0) {
        RowFwdArgs<T> a{};
        a.src0 = static_cast<const T*>(X);
        a.dst0 = static_cast<T*>(Y);
        a.lam = static_cast<const T*>(lam);
        a.lam_mode = (int)lm;
        a.lam_scalar = (T)lam_scalar;
        a.nlines = planes * H;
        a.n = (int)W;
        a.stride = W;
        a.lines_per_plane = H;
        a.C = (int)(C > 0 ? C : 1);
        a.mask_out = mask;
        a.mw = (int)mask_words(W);
        a.ls_after = kLsAfterDefault;
        return cuda_status(launch_row_fwd<T>(a, false, false, s, false), "tv2d_lines_fwd(rows)");
    }
    ColFwdArgs<T> c{};
    c.Z = static_cast<const T*>(X);
    c.Y = static_cast<T*>(Y);
    c.lam = static_cast<const T*>(lam);
    c.lam_mode = (int)lm;
    c.lam_scalar = (T)lam_scalar;
    c.C = (int)(C > 0 ? C : 1);
    c.planes = planes;
    c.H = (int)H;
    c.W = (int)W;
    c.mask_out = mask;
    c.mw = (int)mask_words(H);
    c.ls_after = kLsAfterDefault;
    return cuda_status(launch_col_fwd<T>(c, s, false), "tv2d_lines_fwd(cols)");
}

extern "C" tvp_status_t tv2d_lines_fwd(tvp_dtype_t dt, const void* X, void* Y, int64_t N, int64_t C, int64_t H,
                                       int64_t W, const void* lam, tvp_lam_mode_t lm, double lam_scalar, int axis,
                                       uint32_t* mask, tvp_stream_t stream) {
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv2d_lines_fwd: bad dtype");
    if (!lines_args_ok(N, C, H, W, axis)) return fail(TVP_EINVAL, "tv2d_lines_fwd: need N, C >= 0, H, W >= 1, axis 0/1");
    if (!lam2d_ok(lm, lam, lam_scalar)) return fail(TVP_EINVAL, "tv2d_lines_fwd: invalid lam / lam mode");
    if (N * C == 0) return TVP_OK;
    if (!X || !Y) return fail(TVP_EINVAL, "tv2d_lines_fwd: NULL X or Y");
    if ((axis == 0 ? W : H) > kMaxLine) return fail(TVP_EUNSUPPORTED, "tv2d_lines_fwd: line > tvp_max_line()");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dt == TVP_F32 ? lines_fwd_impl<float>(X, Y, N, C, H, W, lam, lm, lam_scalar, axis, mask, s)
                         : lines_fwd_impl<double>(X, Y, N, C, H, W, lam, lm, lam_scalar, axis, mask, s);
}

template <typename T>
static tvp_status_t lines_bwd_impl(const void* G, const uint32_t* mask, void* GX, void* glam, int64_t N, int64_t C,
                                   int64_t H, int64_t W, tvp_lam_mode_t lm, int axis, void* ws, cudaStream_t s) {
    const int64_t planes = N * C;
    const int64_t L = axis == 0 ? H : W;            // lines per plane
    T* part = static_cast<T*>(ws);
    cudaError_t e;
    if (axis == 0) {
        RowBwdArgs<T> r{};
        r.A = static_cast<const T*>(G);
        r.out = static_cast<T*>(GX);
        r.mask = mask;
        r.mw = (int)mask_words(W);
        r.nlines = planes * H;
        r.n = (int)W;
        r.stride = W;
        r.lam_line = glam ? part : nullptr;
        r.lam_lpp = 1;
        r.lam_pstride = 1;
        e = launch_row_bwd<T>(r, false, false, s);
    } else {
        ColBwdArgs<T> c{};
        c.A = static_cast<const T*>(G);
        c.B = nullptr;
        c.Bout = static_cast<T*>(GX);
        c.mask = mask;
        c.mw = (int)mask_words(H);
        c.planes = planes;
        c.H = (int)H;
        c.W = (int)W;
        c.lam_line = glam ? part : nullptr;
        c.lam_pstride = W;
        e = launch_col_bwd<T>(c, s);
    }
    if (e != cudaSuccess) return cuda_status(e, "tv2d_lines_bwd");
    if (glam) {
        LamReduceArgs<T> q{};
        q.part = part;
        q.out = static_cast<T*>(glam);
        if (lm == TVP_LAM_SCALAR) {
            q.nout = 1; q.reps = 1; q.rep_stride = 0; q.q_stride = 0; q.seglen = planes * L;
        } else if (lm == TVP_LAM_PER_CHANNEL) {
            q.nout = C; q.reps = N; q.rep_stride = C * L; q.q_stride = L; q.seglen = L;
        } else {
            q.nout = planes; q.reps = 1; q.rep_stride = 0; q.q_stride = L; q.seglen = L;
        }
        q.nchunk = lam_chunks(q.reps * q.seglen, q.nout);
        q.scratch = reinterpret_cast<T*>(static_cast<char*>(ws) + align256((size_t)planes * L * sizeof(T)));
        e = launch_lam_reduce<T>(q, s);
    }
    return cuda_status(e, "tv2d_lines_bwd(lam)");
}

extern "C" tvp_status_t tv2d_lines_bwd(tvp_dtype_t dt, const void* grad_Y, const uint32_t* mask, void* grad_X,
                                       void* grad_lam, int64_t N, int64_t C, int64_t H, int64_t W,
                                       tvp_lam_mode_t lm, int axis, void* workspace, tvp_stream_t stream) {
    if (dt != TVP_F32 && dt != TVP_F64) return fail(TVP_EINVAL, "tv2d_lines_bwd: bad dtype");
    if (!lines_args_ok(N, C, H, W, axis)) return fail(TVP_EINVAL, "tv2d_lines_bwd: need N, C >= 0, H, W >= 1, axis 0/1");
    if (lm != TVP_LAM_SCALAR && lm != TVP_LAM_PER_CHANNEL && lm != TVP_LAM_PER_PLANE)
        return fail(TVP_EINVAL, "tv2d_lines_bwd: lam mode must be SCALAR, PER_CHANNEL or PER_PLANE");
    if (N * C == 0) {
        // an empty batch contributes nothing: the lambda gradient is zero (1 or C entries)
        const size_t cnt = lm == TVP_LAM_SCALAR ? 1 : (lm == TVP_LAM_PER_CHANNEL ? (size_t)C : 0);
        if (grad_lam && cnt)
            return cuda_status(cudaMemsetAsync(grad_lam, 0, cnt * (dt == TVP_F64 ? 8 : 4),
                                               reinterpret_cast<cudaStream_t>(stream)), "tv2d_lines_bwd");
        return TVP_OK;
    }
    const int64_t L = axis == 0 ? W : H;
    if (!grad_Y || !grad_X || (L > 1 && !mask)) return fail(TVP_EINVAL, "tv2d_lines_bwd: NULL grad_Y, grad_X or mask");
    if (grad_lam && !workspace) return fail(TVP_EINVAL, "tv2d_lines_bwd: NULL workspace");
    if (L > kMaxLine) return fail(TVP_EUNSUPPORTED, "tv2d_lines_bwd: line > tvp_max_line()");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return dt == TVP_F32 ? lines_bwd_impl<float>(grad_Y, mask, grad_X, grad_lam, N, C, H, W, lm, axis, workspace, s)
                         : lines_bwd_impl<double>(grad_Y, mask, grad_X, grad_lam, N, C, H, W, lm, axis, workspace, s);
}

extern "C" tvp_status_t tvp_softplus_fwd(tvp_dtype_t dt, const void* t, void* lam, int64_t n, tvp_stream_t stream) {
    if ((dt != TVP_F32 && dt != TVP_F64) || n < 0) return fail(TVP_EINVAL, "tvp_softplus_fwd: bad arguments");
    if (n == 0) return TVP_OK;
    if (!t || !lam) return fail(TVP_EINVAL, "tvp_softplus_fwd: NULL pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = dt == TVP_F32 ? launch_softplus<float>((const float*)t, (float*)lam, nullptr, nullptr, n, false, s)
                                  : launch_softplus<double>((const double*)t, (double*)lam, nullptr, nullptr, n, false, s);
    return cuda_status(e, "tvp_softplus_fwd");
}

extern "C" tvp_status_t tvp_softplus_bwd(tvp_dtype_t dt, const void* t, const void* g, void* gt, int64_t n,
                                         tvp_stream_t stream) {
    if ((dt != TVP_F32 && dt != TVP_F64) || n < 0) return fail(TVP_EINVAL, "tvp_softplus_bwd: bad arguments");
    if (n == 0) return TVP_OK;
    if (!t || !g || !gt) return fail(TVP_EINVAL, "tvp_softplus_bwd: NULL pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = dt == TVP_F32 ? launch_softplus<float>((const float*)t, nullptr, (const float*)g, (float*)gt, n, true, s)
                                  : launch_softplus<double>((const double*)t, nullptr, (const double*)g, (double*)gt, n, true, s);
    return cuda_status(e, "tvp_softplus_bwd");
}

extern "C" tvp_status_t tvp_axpby(tvp_dtype_t dt, const void* x, void* y, double a, double b, int64_t n,
                                  tvp_stream_t stream) {
    if ((dt != TVP_F32 && dt != TVP_F64) || n < 0) return fail(TVP_EINVAL, "tvp_axpby: bad arguments");
    if (n == 0) return TVP_OK;
    if (!y || (!x && a != 0.0)) return fail(TVP_EINVAL, "tvp_axpby: NULL pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    cudaError_t e = dt == TVP_F32 ? launch_axpby<float>((const float*)x, (float*)y, (float)a, (float)b, n, s)
                                  : launch_axpby<double>((const double*)x, (double*)y, a, b, n, s);
    return cuda_status(e, "tvp_axpby");
}
