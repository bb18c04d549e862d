// Probe: do shuffles / shared loads eat the same per-SM budget as random global gathers?
// Gather kernel with EXTRA shfl or lds instructions per gather; compare gathers/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 mio_share.cu -o mio_share
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

template <int MODE, int EXTRA>
__global__ void __launch_bounds__(256) gk(const float* __restrict__ x, const int* __restrict__ idx, long long n,
                                          float* out) {
    __shared__ float sm[256 + 8];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    float acc = 0.f;
    const int lane = threadIdx.x & 31;
    int o = lane;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        float v = __ldg(x + __ldg(idx + i));
#pragma unroll
        for (int e = 0; e < EXTRA; e++) {
            if (MODE == 1) v += __shfl_xor_sync(0xffffffffu, v, 1 << (e % 5));
            if (MODE == 2) {
                v += sm[(threadIdx.x & ~31) + ((o + e) & 31)];
            }
        }
        acc += v;
        o = (o + 7) & 31;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

template <int MODE, int EXTRA>
void run(const float* x, const int* idx, long long n, float* out, const char* name) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9f;
    for (int grid : {148 * 8, 148 * 16}) {
        gk<MODE, EXTRA><<<grid, 256>>>(x, idx, n, out);
        cudaEventRecord(a);
        gk<MODE, EXTRA><<<grid, 256>>>(x, idx, n, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    printf("%-6s extra=%2d  %.3f ms  %.1f G gathers/s  %s\n", name, EXTRA, best, n / best / 1e6,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const long long ncols = 1ll << 24, n = 1ll << 26;
    float* x;
    int* idx;
    float* out;
    cudaMalloc(&x, ncols * 4);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 148 * 16 * 256 * 4);
    cudaMemset(x, 0, ncols * 4);
    std::vector<int> h(n);
    unsigned long long s = 42;
    for (long long i = 0; i < n; i++) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        h[i] = (int)((s >> 33) % ncols);
    }
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    run<0, 0>(x, idx, n, out, "plain");
    run<1, 1>(x, idx, n, out, "shfl");
    run<1, 2>(x, idx, n, out, "shfl");
    run<1, 4>(x, idx, n, out, "shfl");
    run<1, 8>(x, idx, n, out, "shfl");
    run<2, 1>(x, idx, n, out, "lds");
    run<2, 2>(x, idx, n, out, "lds");
    run<2, 4>(x, idx, n, out, "lds");
    run<2, 8>(x, idx, n, out, "lds");
    return 0;
}
