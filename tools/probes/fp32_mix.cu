// Does a packed FFMA2 stream (fmaheavy) leave the fmalite pipe free for scalar FFMAs?  Per thread:
// P packed chains + S scalar chains interleaved; reports FP32 lane-ops per clock per SMSP (FFMA2 = 64,
// FFMA = 32 per warp instruction) at the measured SM clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp32_mix.cu -o fp32_mix && ./fp32_mix
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ float ffma3(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
template <int P, int S>
__global__ void kmix(u64* out, u64 a2, u64 b2, float a, float b, int iters) {
    u64 x[P > 0 ? P : 1];
    float y[S > 0 ? S : 1];
    for (int c = 0; c < P; c++) x[c] = threadIdx.x + c;
    for (int c = 0; c < S; c++) y[c] = threadIdx.x + c;
    u64 aa = a2 + threadIdx.x, bb = b2 + threadIdx.x;
    float fa = a + threadIdx.x * 1e-9f, fb = b + threadIdx.x * 1e-9f;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < (P > S ? P : S); c++) {
            if (c < P) x[c] = f2fma(x[c], aa, bb);
            if (c < S) y[c] = ffma3(y[c], fa, fb);
        }
    }
    u64 s = 0;
    for (int c = 0; c < P; c++) s ^= x[c];
    for (int c = 0; c < S; c++) s ^= (u64)__float_as_uint(y[c]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    u64* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz (max)
    const int iters = 20000; float ms;
    auto run = [&](auto kern, int P, int S) {
        kern<<<148 * 8, 256>>>(o, 0x3f8000003f800001ull, 0x3f0000003f000000ull, 1.0001f, 0.5f, iters);
        cudaEventRecord(s); kern<<<148 * 8, 256>>>(o, 0x3f8000003f800001ull, 0x3f0000003f000000ull, 1.0001f, 0.5f, iters);
        cudaEventRecord(e); cudaEventSynchronize(e); cudaEventElapsedTime(&ms, s, e);
        const double warps = 148.0 * 8 * 256 / 32;
        const double ops = warps * iters * (64.0 * P + 32.0 * S);
        const double clocks = ms * 1e-3 * clk * 1e3;
        printf("P=%d S=%d  %.3f ms  %.1f lane-ops/clk/SMSP (at max clock)  instr/clk/SMSP %.3f\n", P, S, ms,
               ops / clocks / 148 / 4, warps * iters * (P + S) / clocks / 148 / 4);
    };
    for (int rep = 0; rep < 2; rep++) {
        run(kmix<8, 0>, 8, 0); run(kmix<0, 8>, 0, 8); run(kmix<4, 4>, 4, 4); run(kmix<4, 8>, 4, 8);
        run(kmix<6, 4>, 6, 4); run(kmix<4, 2>, 4, 2); run(kmix<8, 8>, 8, 8);
    }
    return 0;
}
