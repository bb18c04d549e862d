// Dense BLAS-1/2 PENCIL nests over views: gemv, gemv_t (VOBLA transposed/strided view),
// dot, axpy.  All HBM-bound: the design goal is one pass over the streamed operand with
// 128-bit loads and enough bytes in flight per SM, and no second pass over HBM.
//
// Schedules (from the mapper, see runtime.cpp map_nest):
//   gemv   : i ASSUMED_PARALLEL -> one warp per row;  j PARALLEL_WITH_REDUCTION(+) -> lane-strided
//            partial sums + warp tree.
//   gemv_t : j ASSUMED_PARALLEL -> threads over contiguous columns (coalesced);
//            i PARALLEL_WITH_REDUCTION(+) -> split across CTAs (row blocks), partials reduced
//            in fixed order by the last CTA of each column block (deterministic).
//   dot    : i PARALLEL_WITH_REDUCTION(+) -> grid-stride partials, last-CTA final sum.
//   axpy   : i PARALLEL (AFFINE) -> grid-stride float4 FMA.
#include "common.cuh"
#include "kernels.h"

// ------------------------------------------------------------------ gemv
// A warp owns two rows and streams them together (x loaded once for both): 16 x 16-byte A
// loads in flight per lane.  CTA = 4 warps = 8 rows; at 8192 rows the grid is 1024 CTAs.
// Swept (warps, rows/warp, unroll, CTAs/SM) at 8192^2: (4,2,8,4) 49.2 us, (4,2,4,7) 51.2,
// (4,1,8,8) 51.2, (4,4,4,4) 51.2, (4,4,2,7) 59.4, (8,2,4,3) 59.4.  A pure 268 MB read (dot over
// 2 x 2^25) takes 60.7 us on the same box: at this size the launch ramp and tail, not the
// kernel's streaming rate, set the last ~15%.
#ifndef GEMV_WARPS
#define GEMV_WARPS 4
#endif
#ifndef GEMV_ROWS_PER_WARP
#define GEMV_ROWS_PER_WARP 2
#endif
#ifndef GEMV_UNROLL
#define GEMV_UNROLL 8  // float4 loads per row per lane per iteration
#endif
#ifndef GEMV_MINB
#define GEMV_MINB 4
#endif
template <bool VEC>
__global__ void __launch_bounds__(32 * GEMV_WARPS, GEMV_MINB) gemv_kernel(int m, int n, float alpha, float beta,
                                                                          const float* __restrict__ A,
                                                                          const float* __restrict__ x,
                                                                          float* __restrict__ y) {
    constexpr int R = GEMV_ROWS_PER_WARP, U = GEMV_UNROLL;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long r0 = ((long long)blockIdx.x * GEMV_WARPS + warp) * R;
    if (r0 >= m) return;
    const float* a[R];
#pragma unroll
    for (int r = 0; r < R; r++) a[r] = A + (r0 + r < m ? r0 + r : r0) * (long long)n;  // rows past m: duplicate
    float acc[R][4];
#pragma unroll
    for (int r = 0; r < R; r++) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = 0.f;
    if (VEC) {
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const int n4 = n >> 2;
        int j = lane;
        for (; j + (U - 1) * 32 < n4; j += U * 32) {
            float4 av[R][U], xv[U];
#pragma unroll
            for (int r = 0; r < R; r++)
#pragma unroll
                for (int u = 0; u < U; u++) av[r][u] = ld_stream_f4(reinterpret_cast<const float4*>(a[r]) + j + u * 32);
#pragma unroll
            for (int u = 0; u < U; u++) xv[u] = __ldg(x4 + j + u * 32);
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int r = 0; r < R; r++) {
                    acc[r][0] = fmaf(av[r][u].x, xv[u].x, acc[r][0]);
                    acc[r][1] = fmaf(av[r][u].y, xv[u].y, acc[r][1]);
                    acc[r][2] = fmaf(av[r][u].z, xv[u].z, acc[r][2]);
                    acc[r][3] = fmaf(av[r][u].w, xv[u].w, acc[r][3]);
                }
        }
        for (; j < n4; j += 32) {
            const float4 xv = __ldg(x4 + j);
#pragma unroll
            for (int r = 0; r < R; r++) {
                const float4 v = ld_stream_f4(reinterpret_cast<const float4*>(a[r]) + j);
                acc[r][0] = fmaf(v.x, xv.x, acc[r][0]);
                acc[r][1] = fmaf(v.y, xv.y, acc[r][1]);
                acc[r][2] = fmaf(v.z, xv.z, acc[r][2]);
                acc[r][3] = fmaf(v.w, xv.w, acc[r][3]);
            }
        }
        for (int t = (n4 << 2) + lane; t < n; t += 32) {
            const float xt = __ldg(x + t);
#pragma unroll
            for (int r = 0; r < R; r++) acc[r][0] = fmaf(a[r][t], xt, acc[r][0]);
        }
    } else {
        for (int t = lane; t < n; t += 32) {
            const float xt = __ldg(x + t);
#pragma unroll
            for (int r = 0; r < R; r++) acc[r][0] = fmaf(ld_stream_f(a[r] + t), xt, acc[r][0]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; r++) {
        const float s = warp_sum<32>((acc[r][0] + acc[r][1]) + (acc[r][2] + acc[r][3]));
        if (lane == 0 && r0 + r < m) y[r0 + r] = alpha * s + beta * y[r0 + r];
    }
}

int launch_gemv(cudaStream_t st, int m, int n, float alpha, float beta, const float* A,
                const float* x, float* y) {
    if (m <= 0) return 0;
    bool vec = (n % 4 == 0) && ((uintptr_t)A % 16 == 0) && ((uintptr_t)x % 16 == 0);
    const int rows_per_cta = GEMV_WARPS * GEMV_ROWS_PER_WARP;
    dim3 grid((m + rows_per_cta - 1) / rows_per_cta);
    if (vec) gemv_kernel<true><<<grid, 32 * GEMV_WARPS, 0, st>>>(m, n, alpha, beta, A, x, y);
    else gemv_kernel<false><<<grid, 32 * GEMV_WARPS, 0, st>>>(m, n, alpha, beta, A, x, y);
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ gemv_t
// CTA tile = GT_COLS columns x GT_ROWS rows; 256 threads = 4 row lanes x 64 column lanes,
// each column lane owns 4 adjacent columns (one float4 per row).
#define GT_COLS 256
#define GT_ROWS 256

template <bool VEC>
__global__ void __launch_bounds__(256) gemv_t_kernel(int m, int n, int lda, int incx, int incy,
                                                     float alpha, float beta,
                                                     const float* __restrict__ A,
                                                     const float* __restrict__ x,
                                                     float* __restrict__ y,
                                                     float* __restrict__ partial,
                                                     unsigned* __restrict__ counters) {
    __shared__ float red[4][GT_COLS];
    __shared__ bool is_last;
    const int cl = threadIdx.x & 63, rl = threadIdx.x >> 6;
    const int jb = blockIdx.x, ib = blockIdx.y, nib = gridDim.y;
    const int j0 = jb * GT_COLS + cl * 4;
    const int i_begin = ib * GT_ROWS, i_end = min(m, i_begin + GT_ROWS);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (VEC && j0 + 3 < n) {
        int i = i_begin + rl;
        for (; i + 12 < i_end; i += 16) {
            float4 av[4];
            float xv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                av[u] = ld_stream_f4(reinterpret_cast<const float4*>(A + (long long)(i + 4 * u) * lda + j0));
                xv[u] = __ldg(x + (long long)(i + 4 * u) * incx);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                acc.x = fmaf(av[u].x, xv[u], acc.x);
                acc.y = fmaf(av[u].y, xv[u], acc.y);
                acc.z = fmaf(av[u].z, xv[u], acc.z);
                acc.w = fmaf(av[u].w, xv[u], acc.w);
            }
        }
        for (; i < i_end; i += 4) {
            float4 av = ld_stream_f4(reinterpret_cast<const float4*>(A + (long long)i * lda + j0));
            float xv = __ldg(x + (long long)i * incx);
            acc.x = fmaf(av.x, xv, acc.x);
            acc.y = fmaf(av.y, xv, acc.y);
            acc.z = fmaf(av.z, xv, acc.z);
            acc.w = fmaf(av.w, xv, acc.w);
        }
    } else {
        for (int i = i_begin + rl; i < i_end; i += 4) {
            const float* ar = A + (long long)i * lda;
            float xv = __ldg(x + (long long)i * incx);
            if (j0 + 0 < n) acc.x = fmaf(ld_stream_f(ar + j0 + 0), xv, acc.x);
            if (j0 + 1 < n) acc.y = fmaf(ld_stream_f(ar + j0 + 1), xv, acc.y);
            if (j0 + 2 < n) acc.z = fmaf(ld_stream_f(ar + j0 + 2), xv, acc.z);
            if (j0 + 3 < n) acc.w = fmaf(ld_stream_f(ar + j0 + 3), xv, acc.w);
        }
    }
    red[rl][cl * 4 + 0] = acc.x;
    red[rl][cl * 4 + 1] = acc.y;
    red[rl][cl * 4 + 2] = acc.z;
    red[rl][cl * 4 + 3] = acc.w;
    __syncthreads();
    // fixed-order combine of the 4 row lanes; one column per thread
    const int jc = jb * GT_COLS + threadIdx.x;
    float p = (red[0][threadIdx.x] + red[1][threadIdx.x]) + (red[2][threadIdx.x] + red[3][threadIdx.x]);
    if (nib == 1) {
        if (jc < n) {
            long long iy = (long long)jc * incy;
            y[iy] = alpha * p + beta * y[iy];
        }
        return;
    }
    if (jc < n) partial[(long long)ib * n + jc] = p;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned prev = atomicAdd(&counters[jb], 1u);
        is_last = (prev == (unsigned)nib - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    if (threadIdx.x == 0) counters[jb] = 0;  // self-resetting for the next launch
    if (jc < n) {
        float s = 0.f;
        for (int b = 0; b < nib; b++) s += __ldcg(partial + (long long)b * n + jc);
        long long iy = (long long)jc * incy;
        y[iy] = alpha * s + beta * y[iy];
    }
}

int launch_gemv_t(cudaStream_t st, int m, int n, int lda, int incx, int incy, float alpha,
                  float beta, const float* A, const float* x, float* y, float* partial,
                  unsigned* counters) {
    if (n <= 0) return 0;
    bool vec = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
    int nib = m <= 0 ? 1 : (m + GT_ROWS - 1) / GT_ROWS;
    dim3 grid((n + GT_COLS - 1) / GT_COLS, nib);
    if (vec)
        gemv_t_kernel<true><<<grid, 256, 0, st>>>(m, n, lda, incx, incy, alpha, beta, A, x, y,
                                                  partial, counters);
    else
        gemv_t_kernel<false><<<grid, 256, 0, st>>>(m, n, lda, incx, incy, alpha, beta, A, x, y,
                                                   partial, counters);
    return (int)cudaGetLastError();
}
size_t gemv_t_partial_elems(int m, int n) {
    int nib = m <= 0 ? 1 : (m + GT_ROWS - 1) / GT_ROWS;
    return nib > 1 ? (size_t)nib * (size_t)n : 0;
}
size_t gemv_t_counter_elems(int n) { return (size_t)(n + GT_COLS - 1) / GT_COLS; }

// ------------------------------------------------------------------ dot
#define DOT_BLOCKS (PENCIL_NUM_SMS * 8)
__global__ void __launch_bounds__(256) dot_kernel(long long n, const float* __restrict__ x,
                                                  const float* __restrict__ y,
                                                  float* __restrict__ result,
                                                  double* __restrict__ partial,
                                                  unsigned* __restrict__ counter) {
    __shared__ float wsum[8];
    __shared__ bool is_last;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
    long long done = 0;
    if (vec) {
        const long long n4 = n >> 2;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        const float4* y4 = reinterpret_cast<const float4*>(y);
        long long i = tid;
        for (; i + 3 * nthr < n4; i += 4 * nthr) {
            float4 a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                a[u] = ld_stream_f4(x4 + i + u * nthr);
                b[u] = ld_stream_f4(y4 + i + u * nthr);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                acc0 = fmaf(a[u].x, b[u].x, acc0);
                acc1 = fmaf(a[u].y, b[u].y, acc1);
                acc2 = fmaf(a[u].z, b[u].z, acc2);
                acc3 = fmaf(a[u].w, b[u].w, acc3);
            }
        }
        for (; i < n4; i += nthr) {
            float4 a = ld_stream_f4(x4 + i), b = ld_stream_f4(y4 + i);
            acc0 = fmaf(a.x, b.x, acc0);
            acc1 = fmaf(a.y, b.y, acc1);
            acc2 = fmaf(a.z, b.z, acc2);
            acc3 = fmaf(a.w, b.w, acc3);
        }
        done = n4 << 2;
    }
    for (long long i = done + tid; i < n; i += nthr) acc0 = fmaf(x[i], y[i], acc0);
    float s = warp_sum<32>((acc0 + acc1) + (acc2 + acc3));
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int w = 0; w < 8; w++) b += (double)wsum[w];
        partial[blockIdx.x] = b;
        __threadfence();
        unsigned prev = atomicAdd(counter, 1u);
        is_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // last CTA: fixed-order fp64 sum of the per-CTA partials
    double v = 0.0;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) v += __ldcg(partial + b);
    v = warp_sum_d(v);
    __shared__ double dsum[8];
    if ((threadIdx.x & 31) == 0) dsum[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; w++) t += dsum[w];
        *result = (float)t;
        *counter = 0;
    }
}

int launch_dot(cudaStream_t st, long long n, const float* x, const float* y, float* result,
               double* partial, unsigned* counter) {
    long long want = (n + 4095) / 4096;
    int blocks = (int)(want < DOT_BLOCKS ? (want < 1 ? 1 : want) : DOT_BLOCKS);
    dot_kernel<<<blocks, 256, 0, st>>>(n, x, y, result, partial, counter);
    return (int)cudaGetLastError();
}
size_t dot_partial_elems() { return DOT_BLOCKS; }

// ------------------------------------------------------------------ axpy
// y = a*x + y with the product and the sum each rounded (the emitted C compiled as written):
// bit-identical to the reference CPU path.
__device__ __forceinline__ float axpy1(float a, float x, float y) { return __fadd_rn(__fmul_rn(a, x), y); }

// a_dev != nullptr: the scalar comes from device memory (dot -> axpy chain, no host hop).
__global__ void __launch_bounds__(256) axpy_kernel(long long n, float a_host,
                                                   const float* __restrict__ a_dev,
                                                   const float* __restrict__ x,
                                                   float* __restrict__ y) {
    const float a = a_dev ? __ldg(a_dev) : a_host;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long nthr = (long long)gridDim.x * blockDim.x;
    const bool vec = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0);
    long long done = 0;
    if (vec) {
        const long long n4 = n >> 2;
        const float4* x4 = reinterpret_cast<const float4*>(x);
        float4* y4 = reinterpret_cast<float4*>(y);
        long long i = tid;
        for (; i + 3 * nthr < n4; i += 4 * nthr) {
            float4 xv[4], yv[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                xv[u] = ld_stream_f4(x4 + i + u * nthr);
                yv[u] = ld_stream_f4(reinterpret_cast<const float4*>(y4) + i + u * nthr);
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                float4 r;
                r.x = axpy1(a,xv[u].x, yv[u].x);
                r.y = axpy1(a,xv[u].y, yv[u].y);
                r.z = axpy1(a,xv[u].z, yv[u].z);
                r.w = axpy1(a,xv[u].w, yv[u].w);
                st_stream_f4(y4 + i + u * nthr, r);
            }
        }
        for (; i < n4; i += nthr) {
            float4 xv = ld_stream_f4(x4 + i);
            float4 yv = ld_stream_f4(reinterpret_cast<const float4*>(y4) + i);
            float4 r;
            r.x = axpy1(a,xv.x, yv.x);
            r.y = axpy1(a,xv.y, yv.y);
            r.z = axpy1(a,xv.z, yv.z);
            r.w = axpy1(a,xv.w, yv.w);
            st_stream_f4(y4 + i, r);
        }
        done = n4 << 2;
    }
    for (long long i = done + tid; i < n; i += nthr) y[i] = axpy1(a,x[i], y[i]);
}

int launch_axpy(cudaStream_t st, long long n, float a, const float* a_dev, const float* x,
                float* y) {
    if (n <= 0) return 0;
    long long want = (n + 4095) / 4096;
    int blocks = (int)(want < PENCIL_NUM_SMS * 8 ? want : PENCIL_NUM_SMS * 8);
    axpy_kernel<<<blocks, 256, 0, st>>>(n, a, a_dev, x, y);
    return (int)cudaGetLastError();
}
