// 5x5 image stencils of conv5x5.pencil.c.
//
// Schedule (mapper): i, j ASSUMED_PARALLEL -> 2-D grid of (row band x 128/512-column strip)
// warps; di, dj UNKNOWN -> the 25 taps are folded sequentially per pixel, in source order.
//
// Each warp sweeps DOWN its strip with a 5-row register window: every input row is loaded
// once per strip (128-bit loads, lanes own 4 adjacent pixels — or 16 bytes for packed u8),
// the 2-pixel horizontal halo comes from the neighbour lanes by shuffle and, at the strip
// edges, from one extra load by lanes 0/31.  The only re-read is the 4-row vertical halo
// per band (BAND rows) — 3% extra L2->SM traffic, deduplicated in L2.
//
// conv5x5_f32: interior only, acc = acc + k*img in (di, dj) order, product and sum each rounded
//   to fp32: bit-identical to the reference-emitted C compiled as written.
// conv5x5_u8 (int32 storage, the PENCIL drop-in ABI): clamp-to-edge, int32 multiply-add,
//   (acc + scale/2)/scale truncating, saturate — bit-exact vs the int64 interpreter while
//   |acc| < 2^31 (always for 8-bit images with |k| < 2^18/25... see DESIGN.md).
// conv5x5_u8_bytes (packed u8 storage, 1 B/px): same semantics; taps in int8 range use
//   dp4a: two IDP4A per tap row per pixel with pre-shifted tap words, no byte extraction.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

#define CONV_BAND 64
#define CONV_WARPS 4

struct TapsF { float k[25]; };
struct TapsI { int k[25]; };
// tap words for dp4a: for each kernel row di and output byte slot t (0..3): (lo word, hi word)
struct TapsDp4a { unsigned w[5][4][2]; };

// signed C division (acc + scale/2)/scale, saturated to [0, 255]
struct Divider {
    int scale;
    unsigned long long magic;  // ceil(2^64 / scale) for scale >= 2
};
__device__ __forceinline__ int scale_sat(int acc, const Divider& d) {
    const int half = d.scale / 2;
    if (d.scale > 0) {
        long long nn = (long long)acc + half;
        if (nn < 0) return 0;  // truncation toward zero gives <= 0 -> saturates at 0
        unsigned long long n = (unsigned long long)nn;
        unsigned long long q = d.scale == 1 ? n : __umul64hi(n, d.magic);
        return q > 255ull ? 255 : (int)q;
    }
    int q = (int)(((long long)acc + half) / d.scale);  // rare: negative scale, exact C semantics
    return q < 0 ? 0 : (q > 255 ? 255 : q);
}

// unsigned pixel bytes x signed tap bytes, 32-bit accumulate
__device__ __forceinline__ int dp4a_us(unsigned a, unsigned b, int c) {
    int d;
    asm("dp4a.u32.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ------------------------------------------------------------------ fp32, interior only
// row entry: cols c-2 .. c+5 as r[0..7]
__device__ __forceinline__ void load_row_f32(const float* __restrict__ img, int w, int r, int c,
                                             int lane, float (&e)[8]) {
    const float* row = img + (long long)r * w;
    float4 v;
    if (c + 3 < w) {
        v = ld_stream_f4(reinterpret_cast<const float4*>(row + c));
    } else {
        v.x = c + 0 < w ? row[c + 0] : 0.f;
        v.y = c + 1 < w ? row[c + 1] : 0.f;
        v.z = c + 2 < w ? row[c + 2] : 0.f;
        v.w = c + 3 < w ? row[c + 3] : 0.f;
    }
    float hl0 = 0.f, hl1 = 0.f, hr0 = 0.f, hr1 = 0.f;
    if (lane == 0 && c >= 2) { hl0 = row[c - 2]; hl1 = row[c - 1]; }
    if (lane == 31 && c + 5 < w) { hr0 = row[c + 4]; hr1 = row[c + 5]; }
    float l0 = __shfl_up_sync(0xffffffffu, v.z, 1), l1 = __shfl_up_sync(0xffffffffu, v.w, 1);
    float r0 = __shfl_down_sync(0xffffffffu, v.x, 1), r1 = __shfl_down_sync(0xffffffffu, v.y, 1);
    if (lane == 0) { l0 = hl0; l1 = hl1; }
    if (lane == 31) { r0 = hr0; r1 = hr1; }
    e[0] = l0; e[1] = l1; e[2] = v.x; e[3] = v.y; e[4] = v.z; e[5] = v.w; e[6] = r0; e[7] = r1;
}

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

int launch_conv5x5_f32(cudaStream_t st, int h, int w, const float* img, const float* k25,
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

// ------------------------------------------------------------------ u8 semantics, int32 storage
__device__ __forceinline__ void load_row_i32(const int* __restrict__ img, int h, int w, int r,
                                             int c, int lane, int (&e)[8]) {
    const int* row = img + (long long)clampi(r, 0, h - 1) * w;
    int4 v;
    if (c >= 0 && c + 3 < w) {
        v = ld_stream_i4(reinterpret_cast<const int4*>(row + c));
    } else {
        v.x = row[clampi(c + 0, 0, w - 1)];
        v.y = row[clampi(c + 1, 0, w - 1)];
        v.z = row[clampi(c + 2, 0, w - 1)];
        v.w = row[clampi(c + 3, 0, w - 1)];
    }
    int hl0 = 0, hl1 = 0, hr0 = 0, hr1 = 0;
    if (lane == 0) { hl0 = row[clampi(c - 2, 0, w - 1)]; hl1 = row[clampi(c - 1, 0, w - 1)]; }
    if (lane == 31) { hr0 = row[clampi(c + 4, 0, w - 1)]; hr1 = row[clampi(c + 5, 0, w - 1)]; }
    int l0 = __shfl_up_sync(0xffffffffu, v.z, 1), l1 = __shfl_up_sync(0xffffffffu, v.w, 1);
    int r0 = __shfl_down_sync(0xffffffffu, v.x, 1), r1 = __shfl_down_sync(0xffffffffu, v.y, 1);
    if (lane == 0) { l0 = hl0; l1 = hl1; }
    if (lane == 31) { r0 = hr0; r1 = hr1; }
    e[0] = l0; e[1] = l1; e[2] = v.x; e[3] = v.y; e[4] = v.z; e[5] = v.w; e[6] = r0; e[7] = r1;
}

__global__ void __launch_bounds__(32 * CONV_WARPS) conv5x5_u8_i32_kernel(int h, int w,
                                                                        const int* __restrict__ img,
                                                                        int* __restrict__ out,
                                                                        TapsI k, Divider dv) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * CONV_WARPS + (threadIdx.x >> 5);
    const int c = strip * 128 + lane * 4;
    if (strip * 128 >= w) return;
    const int i0 = blockIdx.y * CONV_BAND;
    const int i1 = min(h, i0 + CONV_BAND);
    int win[5][8];
#pragma unroll
    for (int d = 0; d < 4; d++) load_row_i32(img, h, w, i0 - 2 + d, c, lane, win[d]);
    for (int i = i0; i < i1; i++) {
        load_row_i32(img, h, w, i + 2, c, lane, win[4]);
        int o[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            int acc = 0;
#pragma unroll
            for (int di = 0; di < 5; di++)
#pragma unroll
                for (int dj = 0; dj < 5; dj++) acc += k.k[di * 5 + dj] * win[di][t + dj];
            o[t] = scale_sat(acc, dv);
        }
        int* orow = out + (long long)i * w;
        if (c + 3 < w) {
            *reinterpret_cast<int4*>(orow + c) = make_int4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (c + t < w) orow[c + t] = o[t];
        }
#pragma unroll
        for (int d = 0; d < 4; d++)
#pragma unroll
            for (int q = 0; q < 8; q++) win[d][q] = win[d + 1][q];
    }
}

__global__ void conv5x5_u8_i32_simple(int h, int w, const int* __restrict__ img,
                                      int* __restrict__ out, TapsI k, Divider dv) {
    long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        int i = (int)(p / w), j = (int)(p % w);
        int acc = 0;
        for (int di = 0; di < 5; di++)
            for (int dj = 0; dj < 5; dj++) {
                int r = clampi(i + di - 2, 0, h - 1), cc = clampi(j + dj - 2, 0, w - 1);
                acc += k.k[di * 5 + dj] * __ldg(img + (long long)r * w + cc);
            }
        out[p] = scale_sat(acc, dv);
    }
}

static Divider make_divider(int scale) {
    Divider d;
    d.scale = scale;
    d.magic = 0;
    if (scale >= 2) {
        // ceil(2^64 / scale) = floor((2^64 - 1) / scale) + 1 for every scale >= 2; then
        // floor(n * magic / 2^64) == n / scale exactly while n * scale < 2^64 (n < 2^32 here)
        d.magic = ~0ull / (unsigned long long)scale + 1;
    }
    return d;
}

int launch_conv5x5_u8(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25,
                      int* out) {
    if (h <= 0 || w <= 0) return 0;
    TapsI k;
    for (int t = 0; t < 25; t++) k.k[t] = k25[t];
    Divider dv = make_divider(scale);
    if (w % 4 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0) {
        int strips = (w + 127) / 128;
        dim3 grid((strips + CONV_WARPS - 1) / CONV_WARPS, (h + CONV_BAND - 1) / CONV_BAND);
        conv5x5_u8_i32_kernel<<<grid, 32 * CONV_WARPS, 0, st>>>(h, w, img, out, k, dv);
    } else {
        long long n = (long long)h * w;
        long long blocks = (n + 255) / 256;
        conv5x5_u8_i32_simple<<<(int)(blocks < 65535 ? blocks : 65535), 256, 0, st>>>(h, w, img, out, k, dv);
    }
    return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ packed u8 storage (dp4a)
// A lane owns 16 consecutive pixels = 4 words; the window row keeps 6 words:
// W[0] = bytes c-4..c-1 (from lane-1), W[1..4] own, W[5] = bytes c+16..c+19 (from lane+1).
__device__ __forceinline__ unsigned byte_at_clamped(const unsigned char* row, int w, int x) {
    return row[clampi(x, 0, w - 1)];
}
__device__ __forceinline__ void load_row_u8(const unsigned char* __restrict__ img, int h, int w,
                                            int r, int c, int lane, unsigned (&e)[6]) {
    const unsigned char* row = img + (long long)clampi(r, 0, h - 1) * w;
    uint4 v;
    if (c >= 0 && c + 15 < w) {
        int4 t = ld_stream_i4(reinterpret_cast<const int4*>(row + c));
        v = make_uint4(t.x, t.y, t.z, t.w);
    } else {
        unsigned b[4];
#pragma unroll
        for (int q = 0; q < 4; q++)
            b[q] = byte_at_clamped(row, w, c + 4 * q) | (byte_at_clamped(row, w, c + 4 * q + 1) << 8) |
                   (byte_at_clamped(row, w, c + 4 * q + 2) << 16) | (byte_at_clamped(row, w, c + 4 * q + 3) << 24);
        v = make_uint4(b[0], b[1], b[2], b[3]);
    }
    unsigned hl = 0, hr = 0;
    if (lane == 0)
        hl = byte_at_clamped(row, w, c - 4) | (byte_at_clamped(row, w, c - 3) << 8) |
             (byte_at_clamped(row, w, c - 2) << 16) | (byte_at_clamped(row, w, c - 1) << 24);
    if (lane == 31)
        hr = byte_at_clamped(row, w, c + 16) | (byte_at_clamped(row, w, c + 17) << 8) |
             (byte_at_clamped(row, w, c + 18) << 16) | (byte_at_clamped(row, w, c + 19) << 24);
    unsigned l = __shfl_up_sync(0xffffffffu, v.w, 1);
    unsigned rr = __shfl_down_sync(0xffffffffu, v.x, 1);
    if (lane == 0) l = hl;
    if (lane == 31) rr = hr;
    e[0] = l; e[1] = v.x; e[2] = v.y; e[3] = v.z; e[4] = v.w; e[5] = rr;
}

__global__ void __launch_bounds__(32 * CONV_WARPS) conv5x5_u8_bytes_kernel(
    int h, int w, const unsigned char* __restrict__ img, unsigned char* __restrict__ out,
    TapsDp4a tw, Divider dv) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * CONV_WARPS + (threadIdx.x >> 5);
    const int c = strip * 512 + lane * 16;
    if (strip * 512 >= w) return;
    const int i0 = blockIdx.y * CONV_BAND;
    const int i1 = min(h, i0 + CONV_BAND);
    unsigned win[5][6];
#pragma unroll
    for (int d = 0; d < 4; d++) load_row_u8(img, h, w, i0 - 2 + d, c, lane, win[d]);
    for (int i = i0; i < i1; i++) {
        load_row_u8(img, h, w, i + 2, c, lane, win[4]);
        unsigned packed[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {  // output word q: pixels c+4q .. c+4q+3
            unsigned pw = 0;
#pragma unroll
            for (int t = 0; t < 4; t++) {
                int acc = 0;
#pragma unroll
                for (int di = 0; di < 5; di++) {
                    // t <= 1: bytes span words (q, q+1) of win (win index = word + 1 offset)
                    const unsigned lo = (t <= 1) ? win[di][q] : win[di][q + 1];
                    const unsigned hi = (t <= 1) ? win[di][q + 1] : win[di][q + 2];
                    acc = dp4a_us(lo, tw.w[di][t][0], acc);
                    acc = dp4a_us(hi, tw.w[di][t][1], acc);
                }
                pw |= (unsigned)scale_sat(acc, dv) << (8 * t);
            }
            packed[q] = pw;
        }
        unsigned char* orow = out + (long long)i * w;
        if (c + 15 < w) {
            *reinterpret_cast<uint4*>(orow + c) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
        } else {
#pragma unroll
            for (int q = 0; q < 4; q++)
#pragma unroll
                for (int t = 0; t < 4; t++)
                    if (c + 4 * q + t < w) orow[c + 4 * q + t] = (unsigned char)(packed[q] >> (8 * t));
        }
#pragma unroll
        for (int d = 0; d < 4; d++)
#pragma unroll
            for (int q = 0; q < 6; q++) win[d][q] = win[d + 1][q];
    }
}

__global__ void conv5x5_u8_bytes_simple(int h, int w, const unsigned char* __restrict__ img,
                                        unsigned char* __restrict__ out, TapsI k, Divider dv) {
    long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        int i = (int)(p / w), j = (int)(p % w);
        int acc = 0;
        for (int di = 0; di < 5; di++)
            for (int dj = 0; dj < 5; dj++) {
                int r = clampi(i + di - 2, 0, h - 1), cc = clampi(j + dj - 2, 0, w - 1);
                acc += k.k[di * 5 + dj] * (int)img[(long long)r * w + cc];
            }
        out[p] = (unsigned char)scale_sat(acc, dv);
    }
}

static unsigned pack_s8(int a, int b, int c, int d) {
    return (unsigned)(a & 255) | ((unsigned)(b & 255) << 8) | ((unsigned)(c & 255) << 16) |
           ((unsigned)(d & 255) << 24);
}

int launch_conv5x5_u8_bytes(cudaStream_t st, int h, int w, int scale, const unsigned char* img,
                            const int* k25, unsigned char* out) {
    if (h <= 0 || w <= 0) return 0;
    Divider dv = make_divider(scale);
    bool s8 = true;
    for (int t = 0; t < 25; t++) s8 &= (k25[t] >= -128 && k25[t] <= 127);
    if (s8 && w % 16 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0) {
        TapsDp4a tw;
        for (int di = 0; di < 5; di++) {
            const int* k = k25 + 5 * di;
            // output byte slot t: window bytes j-2..j+2 relative to word q (see kernel)
            tw.w[di][0][0] = pack_s8(0, 0, k[0], k[1]);   // word q-1 bytes 2,3
            tw.w[di][0][1] = pack_s8(k[2], k[3], k[4], 0); // word q   bytes 0..2
            tw.w[di][1][0] = pack_s8(0, 0, 0, k[0]);       // word q-1 byte 3
            tw.w[di][1][1] = pack_s8(k[1], k[2], k[3], k[4]);
            tw.w[di][2][0] = pack_s8(k[0], k[1], k[2], k[3]);  // word q
            tw.w[di][2][1] = pack_s8(k[4], 0, 0, 0);           // word q+1 byte 0
            tw.w[di][3][0] = pack_s8(0, k[0], k[1], k[2]);     // word q bytes 1..3
            tw.w[di][3][1] = pack_s8(k[3], k[4], 0, 0);        // word q+1 bytes 0,1
        }
        int strips = (w + 511) / 512;
        dim3 grid((strips + CONV_WARPS - 1) / CONV_WARPS, (h + CONV_BAND - 1) / CONV_BAND);
        conv5x5_u8_bytes_kernel<<<grid, 32 * CONV_WARPS, 0, st>>>(h, w, img, out, tw, dv);
    } else {
        TapsI k;
        for (int t = 0; t < 25; t++) k.k[t] = k25[t];
        long long n = (long long)h * w;
        long long blocks = (n + 255) / 256;
        conv5x5_u8_bytes_simple<<<(int)(blocks < 65535 ? blocks : 65535), 256, 0, st>>>(h, w, img, out, k, dv);
    }
    return (int)cudaGetLastError();
}
