/*
 * tvprox.h -- C ABI of libtvprox.so, the B200-native (sm_100a) batched TV
 * proximity operators of arXiv 2204.03643 ("Total Variation Optimization
 * Layers for Computer Vision").  Citation keys: P:n = PAPER.md line n.
 *
 * Notation (reading O1/O2): input y, output
 *     x = prox(y, lam) = argmin_x 1/2 ||x - y||^2 + sum_i lam_i |x_{i+1} - x_i|
 * (Eq. 1), D the forward difference (D z)_i = z_{i+1} - z_i, dual
 * u in R^{n-1} with |u_i| <= lam_i (Eq. 5) and x = y - D^T u.
 *
 * Conventions shared by every call
 *  - All data pointers are DEVICE pointers owned by the caller; the library
 *    never allocates, frees or synchronises.  Every call is asynchronous on
 *    `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - dtype selects fp32 or fp64 for I/O and arithmetic.
 *  - Host-detectable argument errors return TVP_EINVAL before any launch;
 *    a launch/driver failure returns TVP_ECUDA (message: tvp_last_error()).
 *    Per-row conditions (non-convergence, non-finite input) never fail a
 *    call; they are reported through row_iters.
 *  - Outputs are bitwise deterministic run to run (no float atomics; all
 *    reductions are fixed-order).
 *  - In-place operation (x == y, Y == X, grad_y == grad_x) is allowed.
 *  - 1D rows may have 1 <= n <= tvp_max_line_1d(dt); 2D rows and columns
 *    1 <= H, W <= tvp_max_line(dt).
 */
#ifndef TVPROX_H_
#define TVPROX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *tvp_stream_t;   /* == cudaStream_t */

typedef enum { TVP_F32 = 0, TVP_F64 = 1 } tvp_dtype_t;

typedef enum {
    TVP_LAM_SCALAR = 0,      /* 1D + 2D: the by-value lam_scalar                      */
    TVP_LAM_PER_ROW = 1,     /* 1D: device T[batch]                                    */
    TVP_LAM_PER_EDGE = 2,    /* 1D: device T[batch][stride], entries 0..n-2 of a row   */
    TVP_LAM_PER_CHANNEL = 3, /* 2D: device T[C] (the TV layer's lambda_c)   */
    TVP_LAM_PER_PLANE = 4    /* 2D: device T[N*C]                                      */
} tvp_lam_mode_t;

typedef enum { TVP_OK = 0, TVP_EINVAL = 1, TVP_EUNSUPPORTED = 2, TVP_ECUDA = 3 } tvp_status_t;

/* row_iters codes written by the forward calls.  A value >= 0 is
 *   bits 0..15   PN iterations,
 *   bit  16      TVP_ITERS_STALL_FLAG: accepted at a rounding-level fixed point,
 *   bits 20..27  line-search passes (function evaluations of the projected line
 *                search of P:188, saturating at 255; 0 when every step was a full
 *                Newton step), see tvp_options_t.
 * (TVP_ITERS_COUNT / TVP_ITERS_LS extract the fields.) */
#define TVP_ITERS_NOT_CONVERGED (-1)   /* max iterations hit; x = y - D^T u (feasible dual) */
#define TVP_ITERS_NONFINITE     (-2)   /* NaN/Inf in the row (or its lam): row set to NaN  */
#define TVP_ITERS_STALL_FLAG    (1 << 16) /* or-ed into a count: accepted at a rounding-level fixed point */
#define TVP_ITERS_COUNT(v)      ((v) & 0xffff)
#define TVP_ITERS_LS(v)         (((v) >> 20) & 0xff)

/* ----------------------------------------------------- per-call options --- */
/*
 * Options of the *_ex calls (NULL = defaults; tvp_options_default fills them).
 * Everything here is per call: no library state is read or written except the
 * calling thread's fused-2D default (tvp_set_fused2d).
 *
 *   fused2d      2D only.  -1: the calling thread's default (initially on, unless
 *                the environment has TVP_FUSED2D=0): planes with 32 < H, W <= 64 run
 *                all K Dykstra passes on chip in one CTA; 0: staged
 *                row / column passes through HBM; 1: on chip wherever supported,
 *                i.e. also fp32 planes whose sides are both in 65..128 or both in
 *                129..224 (C5's 224^2), held by a thread-block cluster of 2-8 CTAs
 *                (distributed shared memory; measured slower than the staged passes
 *                at C5 on B200, so only on request or with TVP_FUSED2D=2).  The
 *                output, saved masks and gradients are bitwise the same either way.
 *   line_search  Globalisation of the projected Newton step:
 *                TVP_LS_BACKTRACK (default) = projected Armijo search with
 *                quadratic-interpolation backtracking ("only iterates a few times",
 *                P:188); TVP_LS_PARALLEL = the parallel multi-step-size search P:188
 *                compares it with (alpha, alpha/2, alpha/4, alpha/8 per pass, the
 *                largest Armijo-accepted one taken).
 *   ls_after     From PN iteration ls_after on, a step whose full Newton point
 *                leaves the box runs the line search; before it, such a step is the
 *                projected full step.  0 = default (12); 1 or 2 = the search guards
 *                every such step (the paper's method as written).  The prox, and so
 *                the result up to rounding, does not depend on it; iteration counts do.
 *   diag         nullable device int32[4], ACCUMULATED by the call (zero it first):
 *                [0] lines solved, [1] lines that ran the line search, [2] line-search
 *                passes, [3] lines accepted at a stall (integer atomics: deterministic).
 *   iter_hist    nullable device int32[passes][TVP_HIST_BINS], ACCUMULATED: number of
 *                lines by PN-iteration count (last bin: not converged or non-finite);
 *                passes = 1 for 1D, 2*iters for 2D (row pass k at 2(k-1), column pass
 *                k at 2(k-1)+1).
 * Errors: TVP_EINVAL for fused2d not in {-1,0,1}, line_search not a
 * tvp_line_search_t, ls_after < 0.
 */
typedef enum { TVP_LS_BACKTRACK = 0, TVP_LS_PARALLEL = 1 } tvp_line_search_t;
#define TVP_HIST_BINS 128
typedef struct tvp_options {
    int fused2d;
    int line_search;
    int ls_after;
    int32_t *diag;
    int32_t *iter_hist;
} tvp_options_t;
void tvp_options_default(tvp_options_t *opts);

/* The calling thread's default for tvp_options_t.fused2d = -1 (thread-local; initially
 * on unless TVP_FUSED2D=0 in the environment).  Returns the previous setting. */
int tvp_set_fused2d(int enable);

/* Longest 2D line (W and H) the register-resident solver takes (1024). */
int64_t tvp_max_line(tvp_dtype_t dt);
/* Longest 1D row (n) ("long 1D signals"): one CTA of up to 16 warps
 * holds a row of up to 8192 (TVP_F32) / 4096 (TVP_F64) samples in registers; longer rows
 * are held by a thread-block cluster of 2..16 such CTAs (distributed shared memory for
 * the solver's scans), up to 65536 samples for both TVP_F32 and TVP_F64. */
int64_t tvp_max_line_1d(tvp_dtype_t dt);

/* ------------------------------------------------------------------ 1D --- */
/*
 * Saved-for-backward mask: 2 bits per edge, edge e (between samples e and
 * e+1) of row b at bits 2*(e%16) of word b*tv1d_mask_words(n) + e/16.
 * Codes: 0 fused (same segment), 1 jump up, 2 jump down, 3 segment boundary
 * with zero jump (only where lam_e = 0; reading O23).  Padding bits are 0.
 * The mask is the support S-bar of D x and its signs.
 */
size_t tv1d_mask_words(int64_t n);                 /* ceil((n-1)/16), 0 if n <= 1 */

/*
 * tv1d_prox_fwd -- batched 1D TV prox (Eq. 1), one problem per row,
 * solved by projected Newton on the dual Eq. 5 with the free-set Newton system
 * Eq. 6 and a projected quadratic-interpolation backtracking line
 * search; duality-gap (KKT) stop test.
 *   y, x        [batch][stride] rows, first n entries used (stride >= n).
 *   lam         TVP_LAM_SCALAR: NULL, value in lam_scalar; PER_ROW: T[batch];
 *               PER_EDGE: T[batch][stride] (entry e = weight of edge e, e < n-1).
 *               lam >= 0; lam = 0 gives x = y bitwise.
 *   mask        nullable; batch*tv1d_mask_words(n) uint32 (needed by the bwd).
 *   row_iters   nullable; int32[batch]: PN iterations, or the TVP_ITERS_ codes.
 * Errors: TVP_EINVAL if y/x NULL (batch > 0), n < 1, batch < 0, stride < n,
 * lam_scalar < 0 or non-finite (SCALAR), lam NULL (other modes), or a 2D
 * mode; TVP_EUNSUPPORTED if n > tvp_max_line_1d(dt).
 */
tvp_status_t tv1d_prox_fwd(tvp_dtype_t dt, const void *y, void *x,
                           int64_t batch, int64_t n, int64_t stride,
                           const void *lam, tvp_lam_mode_t lm, double lam_scalar,
                           uint32_t *mask, int32_t *row_iters, tvp_stream_t stream);

/*
 * tv1d_prox_fwd_warm -- tv1d_prox_fwd whose projected Newton starts from the
 * bound set of a previous solve (DESIGN.md a-11): edges coded up/down in
 * mask_in start bound at +lam/-lam.  The result is the same prox (Eq. 1); only
 * the iteration count changes.  mask_in may alias mask_out (read before write).
 */
tvp_status_t tv1d_prox_fwd_warm(tvp_dtype_t dt, const void *y, void *x,
                                int64_t batch, int64_t n, int64_t stride,
                                const void *lam, tvp_lam_mode_t lm, double lam_scalar,
                                const uint32_t *mask_in, uint32_t *mask_out,
                                int32_t *row_iters, tvp_stream_t stream);

/*
 * tv1d_prox_fwd_ex -- tv1d_prox_fwd (mask_in == NULL) or tv1d_prox_fwd_warm
 * (mask_in != NULL) with per-call options (tvp_options_t; NULL = defaults).
 */
tvp_status_t tv1d_prox_fwd_ex(tvp_dtype_t dt, const void *y, void *x,
                              int64_t batch, int64_t n, int64_t stride,
                              const void *lam, tvp_lam_mode_t lm, double lam_scalar,
                              const uint32_t *mask_in, uint32_t *mask_out, int32_t *row_iters,
                              const tvp_options_t *opts, tvp_stream_t stream);

/* Workspace of tv1d_prox_bwd in bytes (nonzero only for TVP_LAM_SCALAR). */
size_t tv1d_bwd_workspace_bytes(tvp_dtype_t dt, int64_t batch, tvp_lam_mode_t lm);

/*
 * tv1d_prox_bwd -- vector-Jacobian product of tv1d_prox_fwd (Eq. 7-8,
 * P:190-200, reading O12): grad_y = segment-wise mean of grad_x over the
 * segments of the forward's mask; grad_lam from the same segments: a segment
 * [a,b) with boundary signs s_L (edge a-1, 0 at the start) and s_R (edge b-1,
 * 0 at the end) has dx/dlam = (s_R - s_L)/(b-a).
 *   grad_x, grad_y  [batch][stride].
 *   mask            from tv1d_prox_fwd of the same (batch, n).
 *   grad_lam        nullable; SCALAR: T[1] (sum over rows); PER_ROW: T[batch];
 *                   PER_EDGE: T[batch][stride] (e < n-1 written: s_e*(mean_L-mean_R)).
 *   workspace       tv1d_bwd_workspace_bytes(...) bytes (may be NULL if 0).
 */
tvp_status_t tv1d_prox_bwd(tvp_dtype_t dt, const void *grad_x, const uint32_t *mask,
                           void *grad_y, void *grad_lam,
                           int64_t batch, int64_t n, int64_t stride, tvp_lam_mode_t lm,
                           void *workspace, tvp_stream_t stream);

/* ------------------------------------------------------------------ 2D --- */
/*
 * 2D anisotropic TV prox of Eq. 2 per plane of an NCHW tensor,
 * computed as the paper does by `iters` = K iterations of Proximal Dykstra
 * (Algorithm 1; "three or four iterations"), each iteration a
 * row pass then a column pass of the 1D solver above.  One lam is shared by the
 * rows and columns of a plane (reading O4).
 *
 * saved (training), uint32, same 2-bit codes as tv1d: the K row-mask sets
 * [K][N*C][H][ceil((W-1)/16)] (set k-1 = row pass k, line = image row),
 * followed by the K column-mask sets [K][N*C][W][ceil((H-1)/16)] (line = image
 * column, column-major per plane).  Pass k >= 2 of each orientation
 * warm-starts its projected Newton from the mask of pass k-1 (DESIGN.md a-11).
 */
size_t tv2d_saved_bytes(int64_t N, int64_t C, int64_t H, int64_t W, int iters);

/* Workspace (bytes) for tv2d_prox_fwd / tv2d_prox_bwd with these sizes. */
size_t tv2d_workspace_bytes(tvp_dtype_t dt, int64_t N, int64_t C, int64_t H, int64_t W, int iters);

/*
 * tv2d_prox_fwd -- X, Y: contiguous NCHW.  lam per TVP_LAM_SCALAR (lam_scalar),
 * TVP_LAM_PER_CHANNEL (T[C]) or TVP_LAM_PER_PLANE (T[N*C]); lam >= 0.
 * saved nullable (inference).  workspace: tv2d_workspace_bytes(...) bytes.
 * line_iters nullable: int32 [K][2], max PN iterations over the lines of each
 * pass (row, column); a value >= 2^20 means some line of that pass did not
 * converge or was non-finite (diagnostics; written with integer atomics,
 * deterministic).  A non-finite pixel makes its row NaN in row pass 1 and, from
 * there, every line of its plane it reaches; other planes are unaffected.
 * Errors: TVP_EINVAL for NULL X/Y/workspace, N,C < 0, H,W < 1, iters < 1,
 * invalid lam; TVP_EUNSUPPORTED if H or W > tvp_max_line(dt).
 */
tvp_status_t tv2d_prox_fwd(tvp_dtype_t dt, const void *X, void *Y,
                           int64_t N, int64_t C, int64_t H, int64_t W,
                           const void *lam, tvp_lam_mode_t lm, double lam_scalar, int iters,
                           void *saved, void *workspace, int32_t *line_iters,
                           tvp_stream_t stream);

/*
 * tv2d_prox_bwd -- reverse mode through the K unrolled iterations of
 * Algorithm 1, using the masks in `saved` from tv2d_prox_fwd.
 *   grad_Y, grad_X  NCHW.
 *   grad_lam        nullable; SCALAR: T[1]; PER_CHANNEL: T[C]; PER_PLANE: T[N*C].
 *                   (per-process partial sums; a caller sharding N across GPUs
 *                   all-reduces them).
 */
tvp_status_t tv2d_prox_bwd(tvp_dtype_t dt, const void *grad_Y, const void *saved,
                           void *grad_X, void *grad_lam,
                           int64_t N, int64_t C, int64_t H, int64_t W,
                           tvp_lam_mode_t lm, int iters, void *workspace,
                           tvp_stream_t stream);

/* tv2d_prox_fwd / tv2d_prox_bwd with per-call options (tvp_options_t; NULL =
 * defaults).  The backward reads only opts->fused2d. */
tvp_status_t tv2d_prox_fwd_ex(tvp_dtype_t dt, const void *X, void *Y,
                              int64_t N, int64_t C, int64_t H, int64_t W,
                              const void *lam, tvp_lam_mode_t lm, double lam_scalar, int iters,
                              void *saved, void *workspace, int32_t *line_iters,
                              const tvp_options_t *opts, tvp_stream_t stream);
tvp_status_t tv2d_prox_bwd_ex(tvp_dtype_t dt, const void *grad_Y, const void *saved,
                              void *grad_X, void *grad_lam,
                              int64_t N, int64_t C, int64_t H, int64_t W,
                              tvp_lam_mode_t lm, int iters, void *workspace,
                              const tvp_options_t *opts, tvp_stream_t stream);

/* ----------------------------------------------------- TV layer (NEXT f1) --- */
/*
 * The TV layer of Sec. 3.1 (Eq. 3-4, Fig. 2) is built from the calls
 * above plus these.  Rows-only / columns-only spatial modes ("a 1D
 * TV-proximity operator per row or column"): one 1D prox per image row
 * (axis 0, lines of W samples) or image column (axis 1, lines of H samples) of
 * every plane of a contiguous NCHW tensor; lam per TVP_LAM_SCALAR,
 * TVP_LAM_PER_CHANNEL or TVP_LAM_PER_PLANE.  mask (nullable, needed by the
 * bwd): axis 0 [N*C][H][ceil((W-1)/16)], axis 1 [N*C][W][ceil((H-1)/16)].
 */
tvp_status_t tv2d_lines_fwd(tvp_dtype_t dt, const void *X, void *Y,
                            int64_t N, int64_t C, int64_t H, int64_t W,
                            const void *lam, tvp_lam_mode_t lm, double lam_scalar, int axis,
                            uint32_t *mask, tvp_stream_t stream);
size_t tv2d_lines_workspace_bytes(tvp_dtype_t dt, int64_t N, int64_t C, int64_t H, int64_t W, int axis);
tvp_status_t tv2d_lines_bwd(tvp_dtype_t dt, const void *grad_Y, const uint32_t *mask, void *grad_X,
                            void *grad_lam, int64_t N, int64_t C, int64_t H, int64_t W,
                            tvp_lam_mode_t lm, int axis, void *workspace, tvp_stream_t stream);

/* lam = SoftPlus(t) = log(1 + e^t), elementwise over n values (Eq. 3). */
tvp_status_t tvp_softplus_fwd(tvp_dtype_t dt, const void *t, void *lam, int64_t n, tvp_stream_t stream);
/* grad_t = grad_lam * sigmoid(t) (the derivative of SoftPlus). */
tvp_status_t tvp_softplus_bwd(tvp_dtype_t dt, const void *t, const void *grad_lam, void *grad_t,
                              int64_t n, tvp_stream_t stream);
/* y = a*x + b*y over n values (x may be NULL when a == 0; y is not read when
 * b == 0).  Sharpening mode
 * (Eq. 4): Y = 2X - prox(X) is axpby(X, Y_prox, 2, -1); its VJP
 * grad_X = 2G - VJP(G) is axpby(G, VJP(G), 2, -1) and grad_lam is negated. */
tvp_status_t tvp_axpby(tvp_dtype_t dt, const void *x, void *y, double a, double b, int64_t n,
                       tvp_stream_t stream);

/* ------------------------------------------------------------ utilities --- */
const char *tvp_status_string(tvp_status_t s);
const char *tvp_last_error(void);          /* last TVP_ECUDA / TVP_EINVAL message (thread-local) */
int tvp_version(void);                     /* 100 * major + minor */
/* Number of kernel launches issued by this thread since the last reset. */
int64_t tvp_launch_count(int reset);

#ifdef __cplusplus
}
#endif
#endif /* TVPROX_H_ */
