// Throughput probe: FFMA vs FFMA2 (fma.rn.f32x2) vs FMUL+FADD on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma2_rate.cu -o ffma2_rate && ./ffma2_rate
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
template <int CH>
__global__ void k_ffma(float* out, float a, float b, int iters) {
    float x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = fmaf(x[c], a, b);
    float s = 0; for (int c = 0; c < CH; c++) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_ffma2(u64* out, u64 a, u64 b, int iters) {
    u64 x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = f2fma(x[c], a, b);
    u64 s = 0; for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int iters = 20000; float ms;
    for (int rep = 0; rep < 2; rep++) {
    k_ffma<8><<<148 * 8, 256>>>(o, 1.0001f, 0.5f, iters);
    cudaEventRecord(s); k_ffma<8><<<148 * 8, 256>>>(o, 1.0001f, 0.5f, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    double ops = 148.0 * 8 * 256 * iters * 8;
    printf("FFMA : %.1f G lane-ops/s (%.2f per SM-clk at 1.965GHz)\n", ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.965);
    cudaEventRecord(s); k_ffma2<8><<<148 * 8, 256>>>((u64*)o, 0x3f8000003f800000ull, 0x3f0000003f000000ull, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("FFMA2: %.1f G instr-lanes/s = %.1f G fp32 fma/s (%.2f fma per SM-clk)\n", ops / ms / 1e6, 2 * ops / ms / 1e6, 2 * ops / ms / 1e6 / 148 / 1.965);
    }
    return 0;
}
