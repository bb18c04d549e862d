// Shared device helpers for the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PENCIL_NUM_SMS 148

// Device-side fault word (E-INTERP analogue): kernels OR a bit in and keep going; the
// host reads it after the stream synchronizes (runtime.cpp: pencil_sync_status).
enum : unsigned {
    FAULT_OOB_LOAD = 1u,     // load index outside the array (interp.cpp:273-279)
    FAULT_BAD_ROWPTR = 2u,   // CSR rowptr outside [0, nnz]
    FAULT_DIV_ZERO = 4u,     // integer division by zero (interp.cpp:56-57)
};

// L2 eviction-priority policies (createpolicy; the ld .L2::cache_hint operand).
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// Streaming loads: read-only path, no L1 allocation, evict-first from L2 — for data
// touched exactly once (matrix values, CSR arrays, images).
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol_evict_first()));
    return r;
}
__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol_evict_first()));
    return r;
}
__device__ __forceinline__ float ld_stream_f(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(r)
                 : "l"(p), "l"(pol_evict_first()));
    return r;
}
__device__ __forceinline__ int ld_stream_i(const int* p) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(p), "l"(pol_evict_first()));
    return r;
}
__device__ __forceinline__ unsigned ld_stream_u(const unsigned* p) {
    unsigned r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(r)
                 : "l"(p), "l"(pol_evict_first()));
    return r;
}
// A random gather from a vector that L2 should keep (SpMV's x): not allocated in L1, where the
// scattered sectors would only evict lines other warps still need.
__device__ __forceinline__ float ld_gather_f(const float* p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(r)
                 : "l"(p), "l"(pol_evict_last()));
    return r;
}
// Reused data (a gathered vector): keep in L2 as long as possible.
__device__ __forceinline__ float ld_keep_f(const float* p) {
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol_evict_last()));
    return r;
}
__device__ __forceinline__ void st_stream_f4(float4* p, float4 v) {
    asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x),
                 "f"(v.y), "f"(v.z), "f"(v.w));
}

// mbarrier + 1-D bulk async copy (TMA engine, no tensor map): global -> shared, completion
// counted in bytes on the mbarrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "BWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra BWAIT_%=;\n}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
// dst, src 16-byte aligned, bytes a multiple of 16
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

template <int W>
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void raise_fault(unsigned* status, unsigned bit) {
    if (status) atomicOr(status, bit);
}
