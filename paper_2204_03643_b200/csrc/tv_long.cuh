// tv_long.cuh -- f4: 1D rows longer than one CTA holds in registers (SURVEY 8(f) f4,
// north_star "long 1D signals"): one thread-block CLUSTER of NCTA CTAs per row.
//
// Each CTA holds WPL * 32 lanes x E contiguous samples of the row in registers (8192
// fp32 / 4096 fp64 per CTA, as the single-CTA long rows), so a cluster of NCTA = 2..8
// (fp32) / 2..16 (fp64) CTAs holds up to 65536 samples.  The projected-Newton solver
// (pn_solve, Eq. 5-6 in partition form) and the segment-mean backward (Eq. 7-8) are the
// same code as every other path; only their line-group communication is the cluster
// version (CComm, tv_ccomm.cuh): warp aggregates through distributed shared memory and a
// cluster barrier per scan / vote.  Rows are independent problems: each cluster loops
// over rows.  Cold solves start from the empty bound set (the coarse start of the
// shorter rows is per-CTA code and is not used here).
#pragma once
#include "tv_kernels.cuh"
#include "tv_ccomm.cuh"

namespace tvp {

// Dynamic shared memory of the cluster long-row kernels: the CComm slots of the NW warps
// of the cluster, then (forward) the CTA-local Comm slots of its WPL warps and the coarse
// block means of its sub-solve.
template <typename T>
__host__ __device__ constexpr size_t long_comm_bytes(int NW, int WPL = 0) {
    return (size_t)kCommSlots * 3 * NW * sizeof(T) + (size_t)kCommSlots * NW * 4 + (size_t)2 * NW * 4 +
           (size_t)kCommSlots * 3 * WPL * sizeof(T) + (size_t)kCommSlots * WPL * 4 + (size_t)32 * WPL * sizeof(T);
}

// Iteration cap of the cluster-wide solve (the default 64 / 100 is for lines of one CTA:
// rows of 16K-131K samples measured p90 20-28, max 52-54 PN iterations from the
// domain-decomposition start, tools/diag_long.py).
constexpr int kLongMaxIters = 128;

template <typename T, int E, int WPL, int NCTA, bool PE, bool LSP>
__global__ void __launch_bounds__(WPL * 32, 1) k_row_fwd_cl(RowFwdArgs<T> a) {
    static_assert(E % 16 == 0 || 16 % E == 0, "mask words per lane");
    constexpr int NW = WPL * NCTA;
    extern __shared__ __align__(16) unsigned char smraw_[];     // long_comm_bytes<T>(NW)
    T* comm_v = reinterpret_cast<T*>(smraw_);
    int* comm_i = reinterpret_cast<int*>(comm_v + kCommSlots * 3 * NW);
    int* comm_f = comm_i + kCommSlots * NW;
    T* loc_v = reinterpret_cast<T*>(comm_f + 2 * NW);
    int* loc_i = reinterpret_cast<int*>(loc_v + kCommSlots * 3 * WPL);
    T* coarse_v = reinterpret_cast<T*>(loc_i + kCommSlots * WPL);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = (int)cl_rank();
    const CComm<T, WPL, NCTA> C{lane, rank * WPL + warp, comm_v, comm_i, comm_f, smem_u32(comm_v), smem_u32(comm_i),
                               smem_u32(comm_f), 0};
    const Comm<T, 32, WPL> Cl{lane, warp, loc_v, loc_i};   // this CTA alone
    constexpr int PER_CTA = WPL * 32 * E;
    const int ll = (rank * WPL + warp) * 32 + lane;     // line lane
    const int i0 = ll * E;
    const int n = a.n;
    const int nsub = max(0, min(PER_CTA, n - rank * PER_CTA));   // my segment of the row
    const bool vec = ((a.stride & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.src0) | reinterpret_cast<uintptr_t>(a.dst0) |
                       reinterpret_cast<uintptr_t>(PE ? a.lam : a.src0)) & 15) == 0;
    cl_sync();                                          // every CTA of the cluster is running
    for (int64_t r = cl_id(); r < a.nlines; r += cl_num()) {
        T y[E], w[E];
        ld_contig<T, E>(a.src0 + r * a.stride, i0, n, vec, y);
        Lam<T, E, PE> lam;
        if (PE) {
            T le[E];
            ld_contig<T, E>(a.lam + r * a.stride, i0, n - 1, vec, le);
#pragma unroll
            for (int k = 0; k < E; ++k) lam.e[PE ? k : 0] = le[k];
            lam.r = T(0);
        } else {
            lam.r = line_lambda(a.lam, a.lam_mode, a.lam_scalar, r, a.lines_per_plane, a.C);
        }
        uint32_t wp = 0, wn = 0;
        if (a.mask_in && a.mw > 0) {
            uint32_t wb;
            mask_window<E>(a.mask_in + r * a.mw, a.mw, i0, wb, wp, wn);
        } else {
            // Initial bound set (reading O7) by domain decomposition: each CTA first solves
            // its own segment as an independent line (same lambda; the single-CTA solver
            // with its coarse start), and the jumps of that solution start the cluster
            // solve -- they are the global solution's jumps except near the segment cuts,
            // so the cluster-wide iterations only repair the cuts.  Like every warm start
            // this changes iteration counts, not the prox.
            T ys[E], ws[E];
#pragma unroll
            for (int k = 0; k < E; ++k) ys[k] = y[k];
            Lam<T, E, PE> ls = lam;
            solve_line<T, E, 32, WPL, PE, LSP>(ys, ws, ls, nsub, true, 0u, 0u, Cl, a.coarse != 0, coarse_v,
                                               a.ls_after);
            const T wnx = Cl.template next<11>(ws[0]);
            const int e0 = i0 - rank * PER_CTA;
#pragma unroll
            for (int k = 0; k < E; ++k) {
                const T xr = (k + 1 < E) ? ws[(k + 1 < E) ? k + 1 : k] : wnx;
                if (e0 + k < nsub - 1) {
                    wp |= (xr > ws[k] ? 1u : 0u) << k;
                    wn |= (xr < ws[k] ? 1u : 0u) << k;
                }
            }
        }
        const int st = solve_line<T, E, 32, WPL, PE, LSP>(y, w, lam, n, true, wp, wn, C, false, nullptr, a.ls_after,
                                                          kLongMaxIters);
        st_contig<T, E>(a.dst0 + r * a.stride, i0, n, vec, w);
        if (a.mask_out) {
            const T wnext = C.template next<11>(w[0]);
            uint32_t word = 0;
            if constexpr (E == 16 && !PE) {
                word = lane_codes<T, E>(w, wnext, i0, n - 1, !(lam.r > T(0)));
            } else {
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const T xr = (k + 1 < E) ? w[(k + 1 < E) ? k + 1 : k] : wnext;
                    const bool lz = PE ? !(lam.e[PE ? k : 0] > T(0)) : !(lam.r > T(0));
                    const uint32_t code = (i0 + k < n - 1) ? edge_code(w[k], xr, lz) : 0u;
                    word |= code << (2 * ((i0 + k) & 15));
                }
            }
            if (E < 16) {
#pragma unroll
                for (int d = 1; d < 16 / (E < 16 ? E : 16); d <<= 1) word |= __shfl_xor_sync(FULL, word, d);
            }
            const int wd = i0 >> 4;
            if (wd < a.mw && (E >= 16 || (i0 & 15) == 0)) a.mask_out[r * a.mw + wd] = word;
        }
        if (ll == 0) {
            if (a.row_iters) a.row_iters[r] = st;
            if (a.iters_max) atomicMax(a.iters_max, st >= 0 ? (st & 0xffff) : (1 << 20));
            line_diag(st, a.diag, a.hist);
        }
    }
}

template <typename T, int E, int WPL, int NCTA, bool PE>
__global__ void __launch_bounds__(WPL * 32, 1) k_row_bwd_cl(RowBwdArgs<T> a) {
    constexpr int NW = WPL * NCTA;
    extern __shared__ __align__(16) unsigned char smraw_[];     // long_comm_bytes<T>(NW)
    T* comm_v = reinterpret_cast<T*>(smraw_);
    int* comm_i = reinterpret_cast<int*>(comm_v + kCommSlots * 3 * NW);
    int* comm_f = comm_i + kCommSlots * NW;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rank = (int)cl_rank();
    const CComm<T, WPL, NCTA> C{lane, rank * WPL + warp, comm_v, comm_i, comm_f, smem_u32(comm_v), smem_u32(comm_i),
                               smem_u32(comm_f), 0};
    const int ll = (rank * WPL + warp) * 32 + lane;
    const int n = a.n;
    const int i0 = ll * E;
    const bool vec = ((a.stride & 3) == 0) &&
                     ((reinterpret_cast<uintptr_t>(a.out) | reinterpret_cast<uintptr_t>(a.A)) & 15) == 0;
    cl_sync();
    for (int64_t r = cl_id(); r < a.nlines; r += cl_num()) {
        T v[E];
        ld_contig<T, E>(a.A + r * a.stride, i0, n, vec, v);
        uint32_t bnd = 0, pos = 0, neg = 0;
        if (a.mw > 0) mask_window<E>(a.mask + r * a.mw, a.mw, i0, bnd, pos, neg);
        bnd |= pin_tail<E>(n - 1 - i0);
        T lp = T(0);
        seg_mean_c<T, E, 32, WPL>(v, bnd, pos, neg, C, lp);
        if (PE) {
            const T vnx = C.template next<4>(v[0]);
            if (a.lam_edge) {
#pragma unroll
                for (int k = 0; k < E; ++k) {
                    const int e = i0 + k;
                    const T nxt = (k + 1 < E) ? v[(k + 1 < E) ? k + 1 : k] : vnx;
                    if (e < n - 1) {
                        const T sg = bit<E>(pos, k) ? T(1) : (bit<E>(neg, k) ? T(-1) : T(0));
                        a.lam_edge[r * a.stride + e] = sg * (v[k] - nxt);
                    }
                }
            }
        }
        if (a.lam_line) {
            lp = C.template sum<5>(lp);
            if (ll == 0) a.lam_line[(r / a.lam_lpp) * a.lam_pstride + (r % a.lam_lpp)] = lp;
        }
        st_contig<T, E>(a.out + r * a.stride, i0, n, vec, v);
    }
}

}  // namespace tvp
