// Probe: random 16-byte row gathers through the TMA engine (cp.async.bulk.tensor tile::gather4)
// vs the LSU path — can SpMV's x[col] gathers bypass the L1TEX request limit?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_gather4.cu -o tma_gather4
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

#ifndef STAGES
#define STAGES 4
#endif
#ifndef G4_PER_STAGE
#define G4_PER_STAGE 8  // 8 gather4 = 32 rows per stage per warp
#endif
constexpr int WARPS = 4;
#ifndef G4_STRIDE
#define G4_STRIDE 32  // floats between gather4 destinations (TMA wants 128-B aligned smem)
#endif

__global__ void __launch_bounds__(32 * WARPS) g4_kernel(const __grid_constant__ CUtensorMap tm, const int* idx,
                                                        long long nrows_total, float* out) {
    __shared__ __align__(128) float buf[WARPS][STAGES][G4_PER_STAGE * G4_STRIDE];
    __shared__ __align__(8) unsigned long long bar[WARPS][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < STAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long gw = (long long)blockIdx.x * WARPS + warp, nw = (long long)gridDim.x * WARPS;
    const long long per_stage = G4_PER_STAGE * 4;
    const long long nchunks = nrows_total / per_stage;
    float acc = 0.f;
    unsigned phase = 0;
    auto issue = [&](long long ch, int s) {
        const int* ix = idx + ch * per_stage;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[warp][s])),
                     "r"(G4_PER_STAGE * 64)
                     : "memory");
        for (int g = 0; g < G4_PER_STAGE; g++)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], "
                "[%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(&buf[warp][s][g * G4_STRIDE])),
                "l"(&tm), "r"(sa(&bar[warp][s])), "r"(0), "r"(ix[4 * g]), "r"(ix[4 * g + 1]), "r"(ix[4 * g + 2]),
                "r"(ix[4 * g + 3])
                : "memory");
    };
    long long ch = gw;
    int k = 0;
    if (lane == 0)
        for (int s = 0; s < STAGES; s++)
            if (gw + s * nw < nchunks) issue(gw + s * nw, s);
    for (; ch < nchunks; ch += nw, k++) {
        const int s = k % STAGES;
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                sa(&bar[warp][s])),
            "r"((phase >> s) & 1)
            : "memory");
        phase ^= 1u << s;
        acc += buf[warp][s][(lane >> 2) * G4_STRIDE + (lane & 3) * 4];  // one value per gathered row (32 rows per stage)
        __syncwarp();
        if (lane == 0 && ch + STAGES * nw < nchunks) issue(ch + STAGES * nw, s);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

#ifndef LW
#define LW 8
#endif
__global__ void __launch_bounds__(32 * (WARPS + LW)) hyb_kernel(const __grid_constant__ CUtensorMap tm, const int* idx,
                                                               long long n_tma, long long n, const float* x,
                                                               float* out) {
    if (threadIdx.x >= 32 * WARPS) {
        float acc = 0.f;
        const long long t = (long long)blockIdx.x * (32 * LW) + threadIdx.x - 32 * WARPS;
        for (long long i = n_tma + t; i < n; i += (long long)gridDim.x * 32 * LW) acc += x[4ll * idx[i]];
        out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
        return;
    }
    __shared__ __align__(128) float buf[WARPS][STAGES][G4_PER_STAGE * G4_STRIDE];
    __shared__ __align__(8) unsigned long long bar[WARPS][STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int s = 0; s < STAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[warp][s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const long long gw = (long long)blockIdx.x * WARPS + warp, nw = (long long)gridDim.x * WARPS;
    const long long per_stage = G4_PER_STAGE * 4;
    const long long nchunks = n_tma / per_stage;
    float acc = 0.f;
    unsigned phase = 0;
    auto issue = [&](long long ch, int s) {
        const int* ix = idx + ch * per_stage;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[warp][s])),
                     "r"(G4_PER_STAGE * 64)
                     : "memory");
        for (int g = 0; g < G4_PER_STAGE; g++)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], "
                "[%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(sa(&buf[warp][s][g * G4_STRIDE])),
                "l"(&tm), "r"(sa(&bar[warp][s])), "r"(0), "r"(ix[4 * g]), "r"(ix[4 * g + 1]), "r"(ix[4 * g + 2]),
                "r"(ix[4 * g + 3])
                : "memory");
    };
    int k = 0;
    if (lane == 0)
        for (int s = 0; s < STAGES; s++)
            if (gw + s * nw < nchunks) issue(gw + s * nw, s);
    for (long long ch = gw; ch < nchunks; ch += nw, k++) {
        const int s = k % STAGES;
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                sa(&bar[warp][s])),
            "r"((phase >> s) & 1)
            : "memory");
        phase ^= 1u << s;
        acc += buf[warp][s][(lane >> 2) * G4_STRIDE + (lane & 3) * 4];
        __syncwarp();
        if (lane == 0 && ch + STAGES * nw < nchunks) issue(ch + STAGES * nw, s);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void lsu_kernel(const float* x, const int* idx, long long n, float* out) {
    float acc = 0.f;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc += x[4ll * idx[i]];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const long long ncols = 1ll << 24, nrows4 = ncols / 4, n = 1ll << 26;  // 64M row gathers
    float* x;
    int* idx;
    float* out;
    cudaMalloc(&x, ncols * 4);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 148 * 64 * 1024 * 4);
    cudaMemset(x, 0, ncols * 4);
    std::vector<int> h(n);
    unsigned long long s = 42;
    for (long long i = 0; i < n; i++) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = (int)((s >> 33) % nrows4);
    }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {4, (cuuint64_t)nrows4};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)p)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int ctas : {592, 1184, 2368}) {
        g4_kernel<<<ctas, 32 * WARPS>>>(tm, idx, n, out);
        cudaEventRecord(a);
        g4_kernel<<<ctas, 32 * WARPS>>>(tm, idx, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("TMA gather4 ctas=%d: %.3f ms  %.1f G rows/s  err=%s\n", ctas, ms, n / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
    }
    lsu_kernel<<<148 * 8, 256>>>(x, idx, n, out);
    cudaEventRecord(a);
    lsu_kernel<<<148 * 8, 256>>>(x, idx, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("LSU gather: %.3f ms  %.1f G gathers/s\n", ms, n / ms / 1e6);
    for (double f : {0.0, 0.1, 0.2, 0.3})
        for (int ctas : {296, 592, 1184}) {
            long long nt = (long long)(f * n) / 128 * 128;
            hyb_kernel<<<ctas, 32 * (WARPS + LW)>>>(tm, idx, nt, n, x, out);
            cudaEventRecord(a);
            hyb_kernel<<<ctas, 32 * (WARPS + LW)>>>(tm, idx, nt, n, x, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("hybrid f=%.1f ctas=%d: %.3f ms  %.1f G rows/s  err=%s\n", f, ctas, ms, n / ms / 1e6,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
