// Measurement probes (not PENCIL kernels): random-gather rate from a table (the x[col[k]]
// access of SpMV), a float4 copy (HBM roofline check of our own code) and an L2 flush.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

template <int MODE>
__device__ __forceinline__ float gather_ld(const float* p) {
    float r;
    if (MODE == 0) r = *p;
    else if (MODE == 1) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(r) : "l"(p));
    else if (MODE == 2) asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
    else r = ld_keep_f(p);
    return r;
}

// the SpMV data path without rows: stream idx + val (8 B/nnz, 128-bit loads), gather table[idx]
// (the executor's load: evict-last in L2, not allocated in L1), accumulate val * x — the
// practical ceiling of a CSR SpMV on this matrix
__global__ void __launch_bounds__(256) micro_gather_val_kernel(long long n, const int* __restrict__ idx,
                                                               const float* __restrict__ val,
                                                               const float* __restrict__ table,
                                                               float* __restrict__ out) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const long long n4 = n >> 2;
    float acc = 0.f;
    for (long long i = tid; i < n4; i += nthr) {
        const int4 a = ld_stream_i4(reinterpret_cast<const int4*>(idx) + i);
        const float4 v = ld_stream_f4(reinterpret_cast<const float4*>(val) + i);
        acc += v.x * ld_gather_f(table + a.x) + v.y * ld_gather_f(table + a.y) + v.z * ld_gather_f(table + a.z) +
               v.w * ld_gather_f(table + a.w);
    }
    out[tid] = acc;
}

int launch_micro_gather_val(cudaStream_t st, long long n, const int* idx, const float* val, const float* table,
                            float* out) {
    micro_gather_val_kernel<<<PENCIL_NUM_SMS * 8, 256, 0, st>>>(n, idx, val, table, out);
    return (int)cudaGetLastError();
}

template <int MODE>
__global__ void __launch_bounds__(256) micro_gather_kernel(long long n, const int* __restrict__ idx,
                                                           const float* __restrict__ table,
                                                           float* __restrict__ out) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const long long n4 = n >> 2;
    const int4* idx4 = reinterpret_cast<const int4*>(idx);
    float acc = 0.f;
    long long i = tid;
    for (; i + nthr < n4; i += 2 * nthr) {
        int4 a = ld_stream_i4(idx4 + i), b = ld_stream_i4(idx4 + i + nthr);
        acc += gather_ld<MODE>(table + a.x) + gather_ld<MODE>(table + a.y) + gather_ld<MODE>(table + a.z) +
               gather_ld<MODE>(table + a.w) + gather_ld<MODE>(table + b.x) + gather_ld<MODE>(table + b.y) +
               gather_ld<MODE>(table + b.z) + gather_ld<MODE>(table + b.w);
    }
    for (; i < n4; i += nthr) {
        int4 a = ld_stream_i4(idx4 + i);
        acc += gather_ld<MODE>(table + a.x) + gather_ld<MODE>(table + a.y) + gather_ld<MODE>(table + a.z) +
               gather_ld<MODE>(table + a.w);
    }
    out[tid] = acc;
}

// mode bits 0-3: load flavour; 4-7: CTAs per SM (0 -> 8); bit 8: 150 KB dynamic smem per CTA
// (one CTA per SM); bit 9: launch on half the SMs (74 CTAs) — separates per-SM (L1TEX) from
// chip-wide (L2) gather limits.
int launch_micro_gather(cudaStream_t st, int mode, long long n, const int* idx, const float* table,
                        float* out) {
    int per_sm = (mode >> 4) & 15;
    if (!per_sm) per_sm = 8;
    int grid = ((mode >> 9) & 1) ? PENCIL_NUM_SMS / 2 : PENCIL_NUM_SMS * per_sm;
    size_t smem = ((mode >> 8) & 1) ? 150 * 1024 : 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(micro_gather_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(micro_gather_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(micro_gather_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        cudaFuncSetAttribute(micro_gather_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
        attr = true;
    }
    switch (mode & 15) {
        case 0: micro_gather_kernel<0><<<grid, 256, smem, st>>>(n, idx, table, out); break;
        case 1: micro_gather_kernel<1><<<grid, 256, smem, st>>>(n, idx, table, out); break;
        case 2: micro_gather_kernel<2><<<grid, 256, smem, st>>>(n, idx, table, out); break;
        default: micro_gather_kernel<3><<<grid, 256, smem, st>>>(n, idx, table, out); break;
    }
    return (int)cudaGetLastError();
}

__global__ void __launch_bounds__(256) micro_copy_kernel(long long n4, const float4* __restrict__ s,
                                                         float4* __restrict__ d) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    long long i = tid;
    for (; i + 3 * nthr < n4; i += 4 * nthr) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = ld_stream_f4(s + i + u * nthr);
#pragma unroll
        for (int u = 0; u < 4; u++) st_stream_f4(d + i + u * nthr, v[u]);
    }
    for (; i < n4; i += nthr) st_stream_f4(d + i, ld_stream_f4(s + i));
}

int launch_micro_copy(cudaStream_t st, long long n, const float* src, float* dst) {
    micro_copy_kernel<<<PENCIL_NUM_SMS * 8, 256, 0, st>>>(n >> 2, reinterpret_cast<const float4*>(src),
                                                         reinterpret_cast<float4*>(dst));
    return (int)cudaGetLastError();
}

__global__ void micro_fill_kernel(long long n4, float4* __restrict__ d, float v) {
    const long long nthr = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += nthr)
        d[i] = make_float4(v, v, v, v);
}

// Drops the buffer's lines from L2 without writing them back (discard.global.L2, 128 B each).
__global__ void micro_discard_kernel(long long nlines, char* __restrict__ d) {
    const long long nthr = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nlines; i += nthr)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(d + i * 128) : "memory");
}

// L2 flush between timed steps: write the 256 MiB buffer (evicts whatever the last step left),
// then discard its lines, so the next step starts on an empty, CLEAN L2 (as ncu's cache control
// does).  Without the discard ~126 MB of the fill's dirty lines are written back while the next
// step runs (gemv 8192^2: 49.8 us under the fill alone vs 43 us for the kernel itself);
// (-DPENCIL_VARIANT_L2_DIRTY builds the fill-only flush for comparison, tools/variant_build.sh.)
int launch_micro_l2_flush(cudaStream_t st, long long n, float* buf) {
    static float v = 0.f;
#ifdef PENCIL_VARIANT_L2_DIRTY
    const bool dirty = true;
#else
    const bool dirty = false;
#endif
    v += 1.f;
    micro_fill_kernel<<<PENCIL_NUM_SMS * 8, 256, 0, st>>>(n >> 2, reinterpret_cast<float4*>(buf), v);
    if (!dirty) micro_discard_kernel<<<PENCIL_NUM_SMS * 8, 256, 0, st>>>(n * 4 / 128, reinterpret_cast<char*>(buf));
    return (int)cudaGetLastError();
}

