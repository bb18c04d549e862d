// FP32 issue-rate probe on sm_100a: FFMA (3 regs), FMUL / FADD (2 regs), FFMA2 / FMUL2 / FADD2 (packed
// f32x2, 64-bit register pairs).  8 independent chains per thread, 148 x 8 CTAs of 256 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp32_rates.cu -o fp32_rates && ./fp32_rates
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 f2mul(u64 a, u64 b) { u64 r; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ u64 f2add(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float ffma3(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float fmul1(float a, float b) { float r; asm volatile("mul.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fadd1(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
constexpr int CH = 8;
template <int OP>
__global__ void k32(float* out, float a, float b, int iters) {
    float x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    float aa = a + threadIdx.x * 1e-9f, bb = b + threadIdx.x * 1e-9f;  // keep operands in registers
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = OP == 0 ? ffma3(x[c], aa, bb) : OP == 1 ? fmul1(x[c], aa) : fadd1(x[c], bb);
    float s = 0; for (int c = 0; c < CH; c++) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
__global__ void k64(u64* out, u64 a, u64 b, int iters) {
    u64 x[CH];
    for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
    u64 aa = a + threadIdx.x, bb = b + threadIdx.x;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int c = 0; c < CH; c++) x[c] = OP == 0 ? f2fma(x[c], aa, bb) : OP == 1 ? f2mul(x[c], aa) : f2add(x[c], bb);
    u64 s = 0; for (int c = 0; c < CH; c++) s ^= x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
    cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
    const int iters = 20000; float ms;
    const double instr = 148.0 * 8 * 256 * iters * CH / 32;  // warp instructions
    const char* n32[3] = {"FFMA ", "FMUL ", "FADD "};
    const char* n64[3] = {"FFMA2", "FMUL2", "FADD2"};
    for (int rep = 0; rep < 2; rep++) {
        for (int op = 0; op < 3; op++) {
            auto run = [&](auto kern, auto* ptr, auto a, auto b) {
                kern<<<148 * 8, 256>>>(ptr, a, b, iters);
                cudaEventRecord(s); kern<<<148 * 8, 256>>>(ptr, a, b, iters); cudaEventRecord(e); cudaEventSynchronize(e);
                cudaEventElapsedTime(&ms, s, e);
                return instr / (ms * 1e-3) / 148 / 4;  // warp instructions per second per SMSP
            };
            double r32 = op == 0 ? run(k32<0>, o, 1.0001f, 0.5f) : op == 1 ? run(k32<1>, o, 1.0001f, 0.5f) : run(k32<2>, o, 1.0001f, 0.5f);
            u64 a2 = 0x3f8000003f800000ull, b2 = 0x3f0000003f000000ull;
            double r64 = op == 0 ? run(k64<0>, (u64*)o, a2, b2) : op == 1 ? run(k64<1>, (u64*)o, a2, b2) : run(k64<2>, (u64*)o, a2, b2);
            printf("%s %.3f warp-instr/clk/SMSP   %s %.3f warp-instr/clk/SMSP   (at 1.965 GHz)\n", n32[op], r32 / 1.965e9,
                   n64[op], r64 / 1.965e9);
        }
    }
    return 0;
}
