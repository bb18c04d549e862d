// Host -> device from PAGEABLE memory (what a C program relinked from the emitted OpenMP passes):
// the driver's staged copy, page-locking the caller's buffer (cudaHostRegister) around a DMA, and a
// multi-threaded memcpy into pinned staging chunks pipelined with the DMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fopenmp h2d_pageable.cu -o h2d_pageable
#include <cuda_runtime.h>
#include <omp.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main() {
    const size_t N = (size_t)2 << 30;  // 2 GiB
    char* h = (char*)malloc(N);
    #pragma omp parallel for
    for (long long i = 0; i < (long long)N; i += 4096) h[i] = (char)i;
    void* d;
    cudaMalloc(&d, N);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int rep = 0; rep < 2; rep++) {
        double t0 = now();
        cudaMemcpy(d, h, N, cudaMemcpyHostToDevice);
        double t1 = now();
        printf("pageable cudaMemcpy: %.1f GB/s\n", N / (t1 - t0) / 1e9);
        t0 = now();
        cudaHostRegister(h, N, cudaHostRegisterDefault);
        double tr = now();
        cudaMemcpy(d, h, N, cudaMemcpyHostToDevice);
        double tc = now();
        cudaHostUnregister(h);
        t1 = now();
        printf("register %.1f ms + dma %.1f ms + unregister %.1f ms = %.1f GB/s\n", (tr - t0) * 1e3, (tc - tr) * 1e3,
               (t1 - tc) * 1e3, N / (t1 - t0) / 1e9);
        // multi-threaded memcpy into pinned staging, pipelined with the DMA (chunk ring)
        for (int T : {4, 8, 16}) {
            const size_t C = 64 << 20;
            const int R = 4;
            char* st;
            cudaHostAlloc((void**)&st, C * R, cudaHostAllocDefault);
            cudaEvent_t ev[R];
            for (int r = 0; r < R; r++) cudaEventCreateWithFlags(&ev[r], cudaEventDisableTiming);
            // memcpy alone
            t0 = now();
            for (size_t off = 0; off < N; off += C) {
                char* dst = st + ((off / C) % R) * C;
                #pragma omp parallel for num_threads(T)
                for (int t = 0; t < T; t++) memcpy(dst + t * (C / T), h + off + t * (C / T), C / T);
            }
            t1 = now();
            double mc = N / (t1 - t0) / 1e9;
            t0 = now();
            int k = 0;
            for (size_t off = 0; off < N; off += C, k++) {
                const int r = k % R;
                if (k >= R) cudaEventSynchronize(ev[r]);
                char* dst = st + r * C;
                #pragma omp parallel for num_threads(T)
                for (int t = 0; t < T; t++) memcpy(dst + t * (C / T), h + off + t * (C / T), C / T);
                cudaMemcpyAsync((char*)d + off, dst, C, cudaMemcpyHostToDevice, s);
                cudaEventRecord(ev[r], s);
            }
            cudaStreamSynchronize(s);
            t1 = now();
            printf("T=%d: memcpy alone %.1f GB/s, staged pipeline %.1f GB/s\n", T, mc, N / (t1 - t0) / 1e9);
            cudaFreeHost(st);
        }
    }
    return 0;
}
