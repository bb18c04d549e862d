// conv5x5_u8 of conv5x5.pencil.c — 8-bit image semantics, clamp-to-edge borders,
// acc = sum k*img (int), (acc + scale/2)/scale truncating toward zero, saturated to [0, 255].
//
// Integer arithmetic on the fp32 pipe.  With pixels in [0, 255] and |k| <= 657 every partial
// sum is an integer below 2^22, so fp32 FFMA computes it exactly in any order — and the FP32
// pipe is the fast one on sm_100 (128 FMA/clk/SM; measured IDP4A ~16 lane-ops/clk/SM and
// IMAD well below FFMA, tools/probes).  Pixels become floats on entry (int32: OR into the
// 2^23 exponent and subtract; u8: byte_perm into the same pattern), two pixels share one
// packed FFMA2, the sum converts back exactly and the division is a shift (power-of-two scale)
// or a 64-bit magic multiply, both equal to C's truncation on the surviving numerators.
// A warp-row whose window holds a pixel outside [0, 255] (int32 storage is the PENCIL ABI:
// arbitrary ints are legal) or a launch with |k| > 2631 takes the exact int32 path instead.
//
// Layout and traffic: same strip sweep as the fp32 stencil (k_conv.cu) — a lane owns 4
// pixels (int4 for int32 storage, one 32-bit word for packed u8), 5-row register window in
// pair form, 2-row prefetch, unrolled by 10 so window slots are compile-time registers.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int U8_BAND = 64;
constexpr int U8_WARPS = 4;
constexpr int U8_PF = 2;
typedef unsigned long long u64;

struct TapsU8 {
    float k[25];  // exact small integers as fp32 (broadcast from uniform registers)
    int ki[25];   // int taps for the exact fallback
};
struct Div {
    int scale;
    int shift;                 // >= 0: scale == 1 << shift
    unsigned long long magic;  // ceil(2^64 / scale)
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__device__ __forceinline__ unsigned scale_sat(long long acc, const Div& d) {
    if (d.scale > 0) {
        const long long nn = acc + (d.scale >> 1);
        if (nn < 0) return 0u;  // truncation toward zero gives <= 0 -> saturates at 0
        unsigned long long q;
        if (d.shift >= 0) q = (unsigned long long)nn >> d.shift;
        else if (nn >= 256ll * d.scale) return 255u;  // saturates whatever the quotient
        else if (nn < (1ll << 32)) q = __umul64hi((unsigned long long)nn, d.magic);  // n * scale < 2^64
        else q = (unsigned long long)(nn / d.scale);
        return q > 255ull ? 255u : (unsigned)q;
    }
    const long long q = (acc + d.scale / 2) / d.scale;  // negative scale: exact C semantics
    return (unsigned)(q < 0 ? 0 : (q > 255 ? 255 : q));
}

// fast path: |acc| < 2^22; POW2 (scale = 1 << shift, e.g. 1 or 256) stays in 32-bit ints
template <bool POW2>
__device__ __forceinline__ unsigned fast_sat(int acc, const Div& d) {
    if (POW2) {
        const int n = acc + (d.scale >> 1);
        if (n < 0) return 0u;
        const int q = n >> d.shift;
        return q > 255 ? 255u : (unsigned)q;
    }
    return scale_sat(acc, d);
}

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
// exact int -> float for 0 <= v < 2^23
__device__ __forceinline__ float small_i2f(int v) { return __int_as_float(v | 0x4B000000) - 8388608.f; }
// exact float -> int for integer-valued |x| < 2^22 (1.5 * 2^23 shifts it into the mantissa);
// F2I would run on the XU pipe, which saturates first in this kernel
__device__ __forceinline__ int exact_f2i(float x) { return __float_as_int(__fadd_rn(x, 12582912.f)) - 0x4B400000; }

template <bool I32>
struct Pix {
    typedef int T;
};
template <>
struct Pix<false> {
    typedef unsigned char T;
};

// raw row: the lane's 4 pixels + the strip-edge halos of lanes 0 / 31 (2 pixels each side)
template <bool I32>
struct Raw {
    int v[4];
    int hl[2], hr[2];
};

template <bool I32>
__device__ __forceinline__ void issue_row(const typename Pix<I32>::T* __restrict__ img, int h, int w, int r, int c,
                                          int lane, Raw<I32>& rr) {
    const typename Pix<I32>::T* row = img + (long long)clampi(r, 0, h - 1) * w;
    if (c >= 0 && c + 3 < w) {
        if (I32) {
            const int4 v = ld_stream_i4(reinterpret_cast<const int4*>(row + c));
            rr.v[0] = v.x; rr.v[1] = v.y; rr.v[2] = v.z; rr.v[3] = v.w;
        } else {
            const unsigned wd = (unsigned)ld_stream_i(reinterpret_cast<const int*>(row + c));
            rr.v[0] = (int)(wd & 255); rr.v[1] = (int)((wd >> 8) & 255);
            rr.v[2] = (int)((wd >> 16) & 255); rr.v[3] = (int)(wd >> 24);
        }
    } else {
#pragma unroll
        for (int b = 0; b < 4; b++) rr.v[b] = (int)row[clampi(c + b, 0, w - 1)];
    }
    rr.hl[0] = rr.hl[1] = rr.hr[0] = rr.hr[1] = 0;
    if (lane == 0) { rr.hl[0] = (int)row[clampi(c - 2, 0, w - 1)]; rr.hl[1] = (int)row[clampi(c - 1, 0, w - 1)]; }
    if (lane == 31) { rr.hr[0] = (int)row[clampi(c + 4, 0, w - 1)]; rr.hr[1] = (int)row[clampi(c + 5, 0, w - 1)]; }
}

// shuffles + int->float; e[m] = pixel c-2+m; returns whether any of this lane's values is not a byte
template <bool I32>
__device__ __forceinline__ bool finish_row(const Raw<I32>& rr, int lane, u64 (&E)[6]) {
    int l0 = __shfl_up_sync(0xffffffffu, rr.v[2], 1), l1 = __shfl_up_sync(0xffffffffu, rr.v[3], 1);
    int r0 = __shfl_down_sync(0xffffffffu, rr.v[0], 1), r1 = __shfl_down_sync(0xffffffffu, rr.v[1], 1);
    if (lane == 0) { l0 = rr.hl[0]; l1 = rr.hl[1]; }
    if (lane == 31) { r0 = rr.hr[0]; r1 = rr.hr[1]; }
    const int e[8] = {l0, l1, rr.v[0], rr.v[1], rr.v[2], rr.v[3], r0, r1};
    bool bad = false;
    if (I32) bad = ((l0 | l1 | r0 | r1 | rr.v[0] | rr.v[1] | rr.v[2] | rr.v[3]) & ~255) != 0;
    float f[8];
#pragma unroll
    for (int m = 0; m < 8; m++) f[m] = small_i2f(e[m] & 255);
#pragma unroll
    for (int m = 0; m < 6; m++) E[m] = f2pk(f[m], f[m + 2]);  // pixel pairs (t, t+2)
    return bad;
}

template <bool I32>
__device__ __forceinline__ unsigned pixel_exact(const typename Pix<I32>::T* __restrict__ img, int h, int w, int i,
                                                int j, const TapsU8& k, const Div& dv) {
    long long acc = 0;  // int64 like the interpreter (interp.cpp:49-64): exact for any int input
#pragma unroll 1
    for (int di = 0; di < 5; di++) {
        const typename Pix<I32>::T* row = img + (long long)clampi(i + di - 2, 0, h - 1) * w;
#pragma unroll 1
        for (int dj = 0; dj < 5; dj++)
            acc += (long long)k.ki[di * 5 + dj] * (long long)row[clampi(j + dj - 2, 0, w - 1)];
    }
    return scale_sat(acc, dv);
}

template <bool I32>
__device__ __forceinline__ void row_exact(const typename Pix<I32>::T* __restrict__ img, int h, int w, int i, int c,
                                          const TapsU8& k, const Div& dv, unsigned (&o)[4]) {
#pragma unroll
    for (int t = 0; t < 4; t++) o[t] = c + t < w ? pixel_exact<I32>(img, h, w, i, c + t, k, dv) : 0u;
}

template <bool I32, bool POW2, int S, int PR>
__device__ __forceinline__ void u8_step(const typename Pix<I32>::T* __restrict__ img,
                                        typename Pix<I32>::T* __restrict__ out, int h, int w, int i, int c,
                                        int lane, u64 (&W)[5][6], unsigned& badmask, Raw<I32> (&R)[U8_PF],
                                        const TapsU8& k, const Div& dv, bool exact_only) {
    const bool b = finish_row<I32>(R[PR], lane, W[S]);
    badmask = (badmask & ~(1u << S)) | ((unsigned)b << S);
    issue_row<I32>(img, h, w, i + 2 + U8_PF, c, lane, R[PR]);
    unsigned o[4];
    if (!exact_only && !__any_sync(0xffffffffu, badmask != 0)) {
        u64 a02 = 0ull, a13 = 0ull;
#pragma unroll
        for (int di = 0; di < 5; di++) {
            const int sl = (S + 1 + di) % 5;
#pragma unroll
            for (int dj = 0; dj < 5; dj++) {
                const u64 kk = f2pk(k.k[di * 5 + dj], k.k[di * 5 + dj]);
                a02 = f2fma(kk, W[sl][dj], a02);
                a13 = f2fma(kk, W[sl][dj + 1], a13);
            }
        }
        const float2 p02 = f2unpk(a02), p13 = f2unpk(a13);
        o[0] = fast_sat<POW2>(exact_f2i(p02.x), dv);
        o[1] = fast_sat<POW2>(exact_f2i(p13.x), dv);
        o[2] = fast_sat<POW2>(exact_f2i(p02.y), dv);
        o[3] = fast_sat<POW2>(exact_f2i(p13.y), dv);
    } else {
        row_exact<I32>(img, h, w, i, c, k, dv, o);
    }
    typename Pix<I32>::T* orow = out + (long long)i * w;
    if (c + 3 < w) {
        if (I32) *reinterpret_cast<int4*>(orow + c) = make_int4((int)o[0], (int)o[1], (int)o[2], (int)o[3]);
        else *reinterpret_cast<unsigned*>(orow + c) = o[0] | (o[1] << 8) | (o[2] << 16) | (o[3] << 24);
    } else {
#pragma unroll
        for (int t = 0; t < 4; t++)
            if (c + t < w) orow[c + t] = (typename Pix<I32>::T)o[t];
    }
}

template <bool I32, bool POW2>
__global__ void __launch_bounds__(32 * U8_WARPS) conv5x5_u8_kernel(int h, int w,
                                                                   const typename Pix<I32>::T* __restrict__ img,
                                                                   typename Pix<I32>::T* __restrict__ out,
                                                                   TapsU8 k, Div dv, int exact_only) {
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * U8_WARPS + (threadIdx.x >> 5);
    const int c = strip * 128 + lane * 4;
    if (strip * 128 >= w) return;
    const int i0 = blockIdx.y * U8_BAND;
    const int i1 = min(h, i0 + U8_BAND);
    u64 W[5][6];
    unsigned badmask = 0;
    Raw<I32> R[U8_PF];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        Raw<I32> t;
        issue_row<I32>(img, h, w, i0 - 2 + d, c, lane, t);
        badmask |= (unsigned)finish_row<I32>(t, lane, W[d]) << d;
    }
#pragma unroll
    for (int p = 0; p < U8_PF; p++) issue_row<I32>(img, h, w, i0 + 2 + p, c, lane, R[p]);
    for (int i = i0; i < i1; i += 10) {
#define U8_STEP(u) \
    if (i + u < i1) u8_step<I32, POW2, (4 + u) % 5, u % U8_PF>(img, out, h, w, i + u, c, lane, W, badmask, R, k, dv, exact_only != 0);
        U8_STEP(0) U8_STEP(1) U8_STEP(2) U8_STEP(3) U8_STEP(4)
        U8_STEP(5) U8_STEP(6) U8_STEP(7) U8_STEP(8) U8_STEP(9)
#undef U8_STEP
    }
}

template <bool I32>
__global__ void conv5x5_u8_simple(int h, int w, const typename Pix<I32>::T* __restrict__ img,
                                  typename Pix<I32>::T* __restrict__ out, TapsU8 k, Div dv) {
    const long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        out[p] = (typename Pix<I32>::T)pixel_exact<I32>(img, h, w, (int)(p / w), (int)(p % w), k, dv);
}

Div make_div(int scale) {
    Div d;
    d.scale = scale;
    d.shift = -1;
    d.magic = 0;
    if (scale > 0 && (scale & (scale - 1)) == 0) {
        d.shift = 0;
        while ((1 << d.shift) != scale) d.shift++;
    } else if (scale >= 2) {
        d.magic = ~0ull / (unsigned long long)scale + 1;  // ceil(2^64 / scale)
    }
    return d;
}

template <bool I32>
int launch_u8(cudaStream_t st, int h, int w, int scale, const typename Pix<I32>::T* img, const int* k25,
              typename Pix<I32>::T* out) {
    if (h <= 0 || w <= 0) return 0;
    TapsU8 k;
    bool small = true;
    for (int t = 0; t < 25; t++) {
        k.k[t] = (float)k25[t];
        k.ki[t] = k25[t];
        small &= (k25[t] >= -657 && k25[t] <= 657);  // |acc| <= 25 * 255 * 657 < 2^22 (exact_f2i)
    }
    const Div dv = make_div(scale);
    const size_t elem = sizeof(typename Pix<I32>::T);
    if (w % 4 == 0 && (uintptr_t)img % (4 * elem) == 0 && (uintptr_t)out % (4 * elem) == 0) {
        const int strips = (w + 127) / 128;
        dim3 grid((strips + U8_WARPS - 1) / U8_WARPS, (h + U8_BAND - 1) / U8_BAND);
        if (dv.shift >= 0)
            conv5x5_u8_kernel<I32, true><<<grid, 32 * U8_WARPS, 0, st>>>(h, w, img, out, k, dv, small ? 0 : 1);
        else
            conv5x5_u8_kernel<I32, false><<<grid, 32 * U8_WARPS, 0, st>>>(h, w, img, out, k, dv, small ? 0 : 1);
    } else {
        const long long n = (long long)h * w, blocks = (n + 255) / 256;
        conv5x5_u8_simple<I32><<<(int)(blocks < 65535 ? blocks : 65535), 256, 0, st>>>(h, w, img, out, k, dv);
    }
    return (int)cudaGetLastError();
}

}  // namespace

// fallback for layouts the smem-ring kernel (k_stencil.cu) does not take
int launch_conv5x5_u8_reg(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25, int* out) {
    return launch_u8<true>(st, h, w, scale, img, k25, out);
}

// packed-u8 storage through the same fp32 sweep (0.86 ms at 16384^2); the default packed path
// is the dp4a kernel of k_conv_u8b.cu (0.50 ms: 16 px per lane amortise the sweep overhead)
int launch_conv5x5_u8_bytes_fp32(cudaStream_t st, int h, int w, int scale, const unsigned char* img,
                                 const int* k25, unsigned char* out) {
    return launch_u8<false>(st, h, w, scale, img, k25, out);
}
