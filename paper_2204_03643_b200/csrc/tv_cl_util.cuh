// tv_cl_util.cuh -- thread-block-cluster primitives (sm_90+ PTX): CTA rank, cluster id,
// distributed-shared-memory addressing and stores, and the cluster barrier.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvp {

// TVP_CL_COPY (A/B timing builds only): 0 = no exchange, 2 = exchange into the CTA's own
// shared memory (wrong results; isolates the DSMEM cost).  Default 1 = the real exchange.
#ifndef TVP_CL_COPY
#define TVP_CL_COPY 1
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_num() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
// Address of the same shared-memory location in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    if (TVP_CL_COPY == 2) rank = cl_rank();
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// 16-byte store into a (possibly remote) CTA's shared memory.
__device__ __forceinline__ void cl_st4(uint32_t a, float x, float y, float z, float w) {
    if (TVP_CL_COPY == 0) return;
    asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w)
                 : "memory");
}
// 8-byte store into a (possibly remote) CTA's shared memory.
__device__ __forceinline__ void cl_st2(uint32_t a, float x, float y) {
    if (TVP_CL_COPY == 0) return;
    asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
// Scalar stores into a (possibly remote) CTA's shared memory (cluster communication).
__device__ __forceinline__ void cl_put(uint32_t a, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void cl_put(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void cl_put(uint32_t a, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// All threads of all CTAs of the cluster; release / acquire orders the DSMEM stores.
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

}  // namespace tvp
