// Can the GPU read PAGEABLE host memory directly (HMM / ATS: cudaDevAttrPageableMemoryAccess)?
// If so, time a copy kernel reading a malloc'd buffer into device memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmm_probe.cu -o hmm_probe
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
__global__ void pull(const float4* __restrict__ src, float4* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}
int main() {
    int v = 0, v2 = 0, v3 = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0);
    cudaDeviceGetAttribute(&v2, cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
    cudaDeviceGetAttribute(&v3, cudaDevAttrHostRegisterSupported, 0);
    printf("pageableMemoryAccess=%d usesHostPageTables=%d hostRegisterSupported=%d\n", v, v2, v3);
    if (!v) return 0;
    const size_t N = (size_t)1 << 30;
    float* h = (float*)malloc(N);
    for (size_t i = 0; i < N / 4; i += 1024) h[i] = 1.f;
    float* d;
    cudaMalloc(&d, N);
    for (int rep = 0; rep < 3; rep++) {
        auto t0 = std::chrono::steady_clock::now();
        pull<<<148 * 8, 256>>>((const float4*)h, (float4*)d, N / 16);
        cudaError_t e = cudaDeviceSynchronize();
        auto t1 = std::chrono::steady_clock::now();
        double s = std::chrono::duration<double>(t1 - t0).count();
        printf("rep %d: %s %.1f GB/s\n", rep, cudaGetErrorString(e), N / s / 1e9);
    }
    return 0;
}
