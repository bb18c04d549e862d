// conv5x5_f32 of conv5x5.pencil.c: interior-only fp32 5x5 correlation.
//
// Schedule (mapper): i, j ASSUMED_PARALLEL -> 2-D grid of (row band x 128-column strip) warps;
// di, dj UNKNOWN -> the 25 taps are folded sequentially per pixel, in source order, and every
// product and sum rounds to fp32 on its own: bit-identical to the reference-emitted C compiled
// as written.  (conv5x5_u8: k_conv_u8.cu, packed u8: k_conv_u8b.cu.)
//
// Each warp sweeps DOWN its strip with a 5-row register window: every input row is loaded
// once per strip (128-bit loads, a lane owns 4 adjacent pixels), the 2-pixel horizontal halo
// comes from the neighbour lanes by shuffle and, at the strip edges, from one extra load by
// lanes 0/31.  The only re-read is the 4-row vertical halo per band (BAND rows) — 6% extra
// L2->SM traffic, deduplicated in L2.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

#define CONV_BAND 64
#define CONV_WARPS 4

struct TapsF { float k[25]; };
// Packed fp32x2 arithmetic (sm_100 FFMA2): two pixels per instruction.  The as-written
// rounding of `acc += k * img` is kept exactly: p = fma(k, x, -0) rounds the product alone,
// acc = fma(p, 1, acc) rounds the sum alone.  -0 and 1 arrive as kernel parameters so ptxas
// cannot see they are constants (it would otherwise fuse the pair into one FFMA2).
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2pk(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 f2unpk(u64 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
struct TapsF2 {
    float k[25];  // scalar taps: FFMA2 broadcasts a uniform-register scalar to both halves
    u64 negz;     // (-0.0f, -0.0f)
    u64 one;      // (1.0f, 1.0f)
};

// raw row (before the halo shuffles): own float4 + the strip-edge halo loads of lanes 0 / 31
struct RawRow {
    float4 v;
    float hl0, hl1, hr0, hr1;
};
__device__ __forceinline__ void issue_row_f32(const float* __restrict__ img, int w, int r, int c, int lane,
                                              RawRow& rr) {
    const float* row = img + (long long)r * w;
    if (c + 3 < w) {
        rr.v = ld_stream_f4(reinterpret_cast<const float4*>(row + c));
    } else {
        rr.v.x = c + 0 < w ? row[c + 0] : 0.f;
        rr.v.y = c + 1 < w ? row[c + 1] : 0.f;
        rr.v.z = c + 2 < w ? row[c + 2] : 0.f;
        rr.v.w = c + 3 < w ? row[c + 3] : 0.f;
    }
    rr.hl0 = rr.hl1 = rr.hr0 = rr.hr1 = 0.f;
    if (lane == 0 && c >= 2) { rr.hl0 = row[c - 2]; rr.hl1 = row[c - 1]; }
    if (lane == 31 && c + 5 < w) { rr.hr0 = row[c + 4]; rr.hr1 = row[c + 5]; }
}
__device__ __forceinline__ void finish_row_f32(const RawRow& rr, int lane, float (&e)[8]) {
    float l0 = __shfl_up_sync(0xffffffffu, rr.v.z, 1), l1 = __shfl_up_sync(0xffffffffu, rr.v.w, 1);
    float r0 = __shfl_down_sync(0xffffffffu, rr.v.x, 1), r1 = __shfl_down_sync(0xffffffffu, rr.v.y, 1);
    if (lane == 0) { l0 = rr.hl0; l1 = rr.hl1; }
    if (lane == 31) { r0 = rr.hr0; r1 = rr.hr1; }
    e[0] = l0; e[1] = l1; e[2] = rr.v.x; e[3] = rr.v.y; e[4] = rr.v.z; e[5] = rr.v.w; e[6] = r0; e[7] = r1;
}

#define CONV_PF 2  // rows prefetched ahead of the window

// window row in pair form: E[m] = (e[m], e[m+2]), m = 0..5 — lane pixels 0,2 and 1,3 are the
// two halves of the packed accumulators, so tap dj of pixel pair (t, t+2) reads E[t + dj]
__device__ __forceinline__ void pair_row(const float (&e)[8], u64 (&E)[6]) {
#pragma unroll
    for (int m = 0; m < 6; m++) E[m] = f2pk(e[m], e[m + 2]);
}

// One output row.  S = window slot receiving input row i+2; the window rows for di = 0..4 are
// slots (S+1+di) % 5.  PR = raw slot holding row i+2, refilled with row i+2+CONV_PF.
template <int S, int PR>
__device__ __forceinline__ void conv_f32_step(const float* __restrict__ img, float* __restrict__ out, int h,
                                              int w, int i, int c, int lane, u64 (&W)[5][6],
                                              RawRow (&R)[CONV_PF], const TapsF2& k) {
    {
        float e[8];
        finish_row_f32(R[PR], lane, e);
        pair_row(e, W[S]);
    }
    if (i + 2 + CONV_PF < h) issue_row_f32(img, w, i + 2 + CONV_PF, c, lane, R[PR]);
    u64 a02 = 0ull, a13 = 0ull;  // pixels (0, 2) and (1, 3) of the lane
#pragma unroll
    for (int di = 0; di < 5; di++) {
        const int sl = (S + 1 + di) % 5;
#pragma unroll
        for (int dj = 0; dj < 5; dj++) {
            const u64 kk = f2pk(k.k[di * 5 + dj], k.k[di * 5 + dj]);
            a02 = f2fma(f2fma(kk, W[sl][dj], k.negz), k.one, a02);
            a13 = f2fma(f2fma(kk, W[sl][dj + 1], k.negz), k.one, a13);
        }
    }
    const float2 o02 = f2unpk(a02), o13 = f2unpk(a13);
    float* orow = out + (long long)i * w;
    if (c >= 2 && c + 3 < w - 2) {
        st_stream_f4(reinterpret_cast<float4*>(orow + c), make_float4(o02.x, o13.x, o02.y, o13.y));
    } else {
        const float o[4] = {o02.x, o13.x, o02.y, o13.y};
#pragma unroll
        for (int t = 0; t < 4; t++)
            if (c + t >= 2 && c + t < w - 2) orow[c + t] = o[t];
    }
}

__global__ void __launch_bounds__(32 * CONV_WARPS) conv5x5_f32_kernel(int h, int w,
                                                                      const float* __restrict__ img,
                                                                      float* __restrict__ out,
                                                                      TapsF2 k) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * CONV_WARPS + (threadIdx.x >> 5);
    const int c = strip * 128 + lane * 4;
    if (strip * 128 >= w) return;
    const int i0 = 2 + blockIdx.y * CONV_BAND;
    const int i1 = min(h - 2, i0 + CONV_BAND);
    if (i0 >= i1) return;
    u64 W[5][6];
    RawRow R[CONV_PF];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        RawRow t;
        float e[8];
        issue_row_f32(img, w, i0 - 2 + d, c, lane, t);
        finish_row_f32(t, lane, e);
        pair_row(e, W[d]);
    }
#pragma unroll
    for (int p = 0; p < CONV_PF; p++)
        if (i0 + 2 + p < h) issue_row_f32(img, w, i0 + 2 + p, c, lane, R[p]);
    // 10 = lcm(5 window slots, 2 raw slots): every slot index is a compile-time constant
    for (int i = i0; i < i1; i += 10) {
#define CONV_F32_STEP(u) \
    if (i + u < i1) conv_f32_step<(4 + u) % 5, u % CONV_PF>(img, out, h, w, i + u, c, lane, W, R, k);
        CONV_F32_STEP(0) CONV_F32_STEP(1) CONV_F32_STEP(2) CONV_F32_STEP(3) CONV_F32_STEP(4)
        CONV_F32_STEP(5) CONV_F32_STEP(6) CONV_F32_STEP(7) CONV_F32_STEP(8) CONV_F32_STEP(9)
#undef CONV_F32_STEP
    }
}

// scalar fallback for unaligned layouts (w % 4 != 0 or misaligned base)
__global__ void conv5x5_f32_simple(int h, int w, const float* __restrict__ img,
                                   float* __restrict__ out, TapsF k) {
    long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        int i = (int)(p / w), j = (int)(p % w);
        if (i < 2 || i >= h - 2 || j < 2 || j >= w - 2) continue;
        float acc = 0.f;
        for (int di = 0; di < 5; di++)
            for (int dj = 0; dj < 5; dj++)
                acc = __fadd_rn(acc, __fmul_rn(k.k[di * 5 + dj], __ldg(img + (long long)(i + di - 2) * w + (j + dj - 2))));
        out[p] = acc;
    }
}

// fallback for layouts the smem-ring kernel (k_stencil.cu) does not take
int launch_conv5x5_f32_reg(cudaStream_t st, int h, int w, const float* img, const float* k25,
                           float* out) {
    if (h < 5 || w < 5) return 0;
    TapsF k;
    for (int t = 0; t < 25; t++) k.k[t] = k25[t];
    if (w % 4 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0) {
        TapsF2 k2;
        auto pack2 = [](float v) {
            unsigned u;
            memcpy(&u, &v, 4);
            return ((unsigned long long)u << 32) | u;
        };
        for (int t = 0; t < 25; t++) k2.k[t] = k25[t];
        k2.negz = pack2(-0.0f);
        k2.one = pack2(1.0f);
        int strips = (w + 127) / 128;
        dim3 grid((strips + CONV_WARPS - 1) / CONV_WARPS, (h - 4 + CONV_BAND - 1) / CONV_BAND);
        conv5x5_f32_kernel<<<grid, 32 * CONV_WARPS, 0, st>>>(h, w, img, out, k2);
    } else {
        long long n = (long long)h * w;
        long long blocks = (n + 255) / 256;
        conv5x5_f32_simple<<<(int)(blocks < 65535 ? blocks : 65535), 256, 0, st>>>(h, w, img, out, k);
    }
    return (int)cudaGetLastError();
}

