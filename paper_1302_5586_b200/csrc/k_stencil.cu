// 5x5 stencils (conv5x5.pencil.c) — the default path for 16-byte-aligned images with w % 4 == 0.
//
// The register-window sweeps of k_conv.cu / k_conv_u8.cu held their prefetched rows in
// registers (~120 registers, 16 warps per SM): too few bytes in flight for HBM, latency-bound
// at 0.67 / 0.77 ms.  Here every warp streams its 128-column strip through a private 8-row
// shared-memory ring filled by cp.async (16 B per lane + 16-byte halo words from lanes 0/31),
// so 7 rows per warp are in flight without holding registers; a row is read once from smem
// into the 5-row register window (packed pixel pairs for FFMA2) when it enters it, and its ring
// slot is refilled at once.  Window slots rotate at compile time (unroll by 5).
//
// Policies (same arithmetic as the fallbacks, so the parity claims carry over unchanged):
//   F32  conv5x5_f32: interior only; acc = acc + k*img per tap in source order with the product
//        and the sum each rounded (FFMA2 against runtime -0 / 1): bit-exact vs the emitted C.
//   U8   conv5x5_u8 on int32 storage: clamp-to-edge; integer sums on the fp32 pipe (exact for
//        pixels in [0, 255] and |k| <= 657); a warp-row whose window holds a non-byte value (or
//        a launch with larger taps) takes the exact int64 path from global memory.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int S_WARPS = 4;
constexpr int S_BAND = 64;
constexpr int S_RING = 8;    // rows per warp ring
constexpr int S_ROWE = 136;  // ring row: columns [c0 - 4, c0 + 132)
typedef unsigned long long u64;

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
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
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct StencilArgs {
    float kf[25];              // taps as fp32 (exact small integers for U8)
    long long ki[25];          // int taps for the exact U8 path
    u64 negz, one;             // runtime (-0, -0) and (1, 1) for the F32 exact rounding
    int scale, shift;          // U8: scale, shift >= 0 when scale = 1 << shift
    unsigned long long magic;  // U8: ceil(2^64 / scale)
    int exact_only;            // U8: taps too large for the fp32 path
    unsigned* repair_flag;     // U8: set when some window held a value outside [0, 255]
};

__device__ __forceinline__ unsigned sat_div(long long acc, const StencilArgs& a) {
    if (a.scale > 0) {
        const long long nn = acc + (a.scale >> 1);
        if (nn < 0) return 0u;
        if (a.shift >= 0) {
            const long long q = nn >> a.shift;
            return q > 255 ? 255u : (unsigned)q;
        }
        if (nn >= 256ll * a.scale) return 255u;
        const unsigned long long q = nn < (1ll << 32) ? __umul64hi((unsigned long long)nn, a.magic)
                                                      : (unsigned long long)(nn / a.scale);
        return q > 255ull ? 255u : (unsigned)q;
    }
    const long long q = (acc + a.scale / 2) / a.scale;
    return (unsigned)(q < 0 ? 0 : (q > 255 ? 255 : q));
}

template <bool U8>
struct Pol {
    typedef float T;
};
template <>
struct Pol<true> {
    typedef int T;
};

template <bool U8>
__device__ __forceinline__ void ring_issue(const typename Pol<U8>::T* __restrict__ img, int h, int w, int r, int c0,
                                           int lane, typename Pol<U8>::T* slot) {
    const int rr = U8 ? clampi(r, 0, h - 1) : r;
    const typename Pol<U8>::T* src = img + (long long)rr * w;
    const int c = c0 + 4 * lane;
    if (c + 3 < w) cp16(slot + 4 + 4 * lane, src + c);
    if (lane == 0 && c0 >= 4) cp16(slot, src + c0 - 4);
    if (lane == 31 && c0 + 131 < w) cp16(slot + 132, src + c0 + 128);
}

// window row entering the register window: pixel pairs E[m] = (e[m], e[m+2]), e[m] = column
// c-2+m (clamped for U8); returns whether any value is outside [0, 255] (U8)
template <bool U8>
__device__ __forceinline__ bool ring_read(const typename Pol<U8>::T* slot, int w, int c0, int lane, u64 (&E)[6]) {
    const int c = c0 + 4 * lane;
    // columns c-2 .. c+5 sit at ring index 4*lane+2 .. 4*lane+9: 8 B + 16 B + 8 B aligned reads
    typename Pol<U8>::T v[8];
    const typename Pol<U8>::T* p = slot + 4 * lane + 2;
    {
        const uint2 l = *reinterpret_cast<const uint2*>(p);
        const uint4 mid = *reinterpret_cast<const uint4*>(p + 2);
        const uint2 r = *reinterpret_cast<const uint2*>(p + 6);
        const unsigned u[8] = {l.x, l.y, mid.x, mid.y, mid.z, mid.w, r.x, r.y};
#pragma unroll
        for (int m = 0; m < 8; m++) memcpy(&v[m], &u[m], 4);
    }
    if (U8 && (c0 == 0 || c0 + 132 > w)) {  // image-edge strips: clamp-to-edge columns
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const int col = c - 2 + m;
            if (col < 0 || col > w - 1) v[m] = slot[clampi(col, 0, w - 1) - (c0 - 4)];
        }
    }
    float f[8];
    bool bad = false;
    if (U8) {
        int orv = 0;
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const int iv = (int)v[m];
            orv |= iv;
            f[m] = __int_as_float((iv & 255) | 0x4B000000) - 8388608.f;  // exact int -> float
        }
        bad = (orv & ~255) != 0;
    } else {
#pragma unroll
        for (int m = 0; m < 8; m++) f[m] = (float)v[m];
    }
#pragma unroll
    for (int m = 0; m < 6; m++) E[m] = f2pk(f[m], f[m + 2]);
    return bad;
}

template <bool U8>
__device__ __forceinline__ unsigned pixel_exact(const int* __restrict__ img, int h, int w, int i, int j,
                                                const StencilArgs& a) {
    long long acc = 0;
#pragma unroll 1
    for (int di = 0; di < 5; di++) {
        const int* row = img + (long long)clampi(i + di - 2, 0, h - 1) * w;
#pragma unroll 1
        for (int dj = 0; dj < 5; dj++) acc += a.ki[di * 5 + dj] * (long long)row[clampi(j + dj - 2, 0, w - 1)];
    }
    return sat_div(acc, a);
}

template <bool U8, int S, bool POW2>
__device__ __forceinline__ void stencil_step(const typename Pol<U8>::T* __restrict__ img,
                                             typename Pol<U8>::T* __restrict__ out, int h, int w, int i, int c0,
                                             int lane, int r_end, typename Pol<U8>::T (*ring)[S_ROWE], u64 (&W)[5][6],
                                             unsigned& badmask, const StencilArgs& a) {
    // the ring holds rows i+2 .. i+2+S_RING-1 in flight; the oldest (row i+2) must have landed
    cp_wait<S_RING - 1>();
    __syncwarp();
    typename Pol<U8>::T* slot = ring[(i + 2) % S_RING];
    const bool b = ring_read<U8>(slot, w, c0, lane, W[S]);
    if (U8) badmask = (badmask & ~(1u << S)) | ((unsigned)b << S);
    __syncwarp();
    if (i + 2 + S_RING < r_end) ring_issue<U8>(img, h, w, i + 2 + S_RING, c0, lane, slot);
    cp_commit();

    const int c = c0 + 4 * lane;
    float o[4];
    // a non-byte pixel in the window: flag the launch for the exact repair pass (u8_repair_kernel)
    // and keep going — keeping the exact path out of this loop keeps it at 80 registers
    if (U8 && __any_sync(0xffffffffu, badmask != 0) && lane == 0) atomicOr(a.repair_flag, 1u);
    const bool exact = false;
    if (!exact) {
        u64 a02 = 0ull, a13 = 0ull;
#pragma unroll
        for (int di = 0; di < 5; di++) {
            const int sl = (S + 1 + di) % 5;
#pragma unroll
            for (int dj = 0; dj < 5; dj++) {
                const u64 kk = f2pk(a.kf[di * 5 + dj], a.kf[di * 5 + dj]);
                if (U8) {  // exact integer sums: fused is fine
                    a02 = f2fma(kk, W[sl][dj], a02);
                    a13 = f2fma(kk, W[sl][dj + 1], a13);
                } else {   // product and sum rounded separately, as written
                    a02 = f2fma(f2fma(kk, W[sl][dj], a.negz), a.one, a02);
                    a13 = f2fma(f2fma(kk, W[sl][dj + 1], a.negz), a.one, a13);
                }
            }
        }
        const float2 p02 = f2unpk(a02), p13 = f2unpk(a13);
        o[0] = p02.x; o[1] = p13.x; o[2] = p02.y; o[3] = p13.y;
    }
    typename Pol<U8>::T* orow = out + (long long)i * w;
    if (U8) {
        int v[4];
        if (!exact) {
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int acc = __float_as_int(__fadd_rn(o[t], 12582912.f)) - 0x4B400000;  // exact, |acc| < 2^22
                if (POW2) {
                    const int n = acc + (a.scale >> 1);
                    v[t] = n < 0 ? 0 : min(n >> a.shift, 255);
                } else {
                    v[t] = (int)sat_div(acc, a);
                }
            }
        }
        if (c + 3 < w) *reinterpret_cast<int4*>((int*)orow + c) = make_int4(v[0], v[1], v[2], v[3]);
        else
            for (int t = 0; t < 4; t++)
                if (c + t < w) ((int*)orow)[c + t] = v[t];
    } else {
        if (c >= 2 && c + 3 < w - 2) {
            st_stream_f4(reinterpret_cast<float4*>((float*)orow + c), make_float4(o[0], o[1], o[2], o[3]));
        } else {
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (c + t >= 2 && c + t < w - 2) ((float*)orow)[c + t] = o[t];
        }
    }
}

template <bool U8, bool POW2>
__global__ void __launch_bounds__(32 * S_WARPS, U8 ? 5 : 6) stencil_ring_kernel(int h, int w,
                                                                       const typename Pol<U8>::T* __restrict__ img,
                                                                       typename Pol<U8>::T* __restrict__ out,
                                                                       StencilArgs a) {
    __shared__ __align__(16) typename Pol<U8>::T ring_all[S_WARPS][S_RING][S_ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int strip = blockIdx.x * S_WARPS + warp;
    const int c0 = strip * 128;
    if (c0 >= w) return;
    // output rows [i0, i1); input rows [i0 - 2, i1 + 2)
    const int i0 = (U8 ? 0 : 2) + blockIdx.y * S_BAND;
    const int i1 = min(U8 ? h : h - 2, i0 + S_BAND);
    if (i0 >= i1) return;
    const int r_end = i1 + 2;
    typename Pol<U8>::T(*ring)[S_ROWE] = ring_all[warp];
#pragma unroll
    for (int d = 0; d < S_RING; d++) {  // prologue: rows i0-2 .. i0+5 in flight
        if (i0 - 2 + d < r_end) ring_issue<U8>(img, h, w, i0 - 2 + d, c0, lane, ring[(i0 - 2 + d + S_RING) % S_RING]);
        cp_commit();
    }
    u64 W[5][6];
    unsigned badmask = 0;
#pragma unroll
    for (int d = 0; d < 4; d++) {  // rows i0-2 .. i0+1 into the window, slots refilled
        cp_wait<S_RING - 1>();
        __syncwarp();
        typename Pol<U8>::T* slot = ring[(i0 - 2 + d + S_RING) % S_RING];
        const bool b = ring_read<U8>(slot, w, c0, lane, W[d]);
        if (U8) badmask |= (unsigned)b << d;
        __syncwarp();
        if (i0 - 2 + d + S_RING < r_end) ring_issue<U8>(img, h, w, i0 - 2 + d + S_RING, c0, lane, slot);
        cp_commit();
    }
    for (int i = i0; i < i1; i += 5) {
        stencil_step<U8, 4, POW2>(img, out, h, w, i, c0, lane, r_end, ring, W, badmask, a);
        if (i + 1 < i1) stencil_step<U8, 0, POW2>(img, out, h, w, i + 1, c0, lane, r_end, ring, W, badmask, a);
        if (i + 2 < i1) stencil_step<U8, 1, POW2>(img, out, h, w, i + 2, c0, lane, r_end, ring, W, badmask, a);
        if (i + 3 < i1) stencil_step<U8, 2, POW2>(img, out, h, w, i + 3, c0, lane, r_end, ring, W, badmask, a);
        if (i + 4 < i1) stencil_step<U8, 3, POW2>(img, out, h, w, i + 4, c0, lane, r_end, ring, W, badmask, a);
    }
    cp_wait<0>();
}

// exact int64 repair pass for conv5x5_u8 on int32 storage: runs after the fast kernel and
// exits at once unless that kernel flagged a non-byte pixel (or the taps are too large for the
// fp32 path); then it recomputes every pixel exactly and re-arms the flag.
__global__ void u8_repair_kernel(int h, int w, const int* __restrict__ img, int* __restrict__ out,
                                 StencilArgs a) {
    if (!a.exact_only && *(volatile unsigned*)a.repair_flag == 0) return;
    const long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x)
        out[p] = (int)pixel_exact<true>(img, h, w, (int)(p / w), (int)(p % w), a);
}
__global__ void u8_rearm_kernel(unsigned* flag) { *flag = 0u; }

u64 pack2(float v) {
    unsigned u;
    memcpy(&u, &v, 4);
    return ((u64)u << 32) | u;
}

bool ring_ok(int h, int w, const void* img, const void* out) {
    return h >= 1 && w >= 4 && w % 4 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0;
}

}  // namespace

// fallbacks (register-window sweeps and scalar kernels) for other layouts
int launch_conv5x5_f32_reg(cudaStream_t st, int h, int w, const float* img, const float* k25, float* out);
int launch_conv5x5_u8_reg(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25, int* out);

int launch_conv5x5_f32(cudaStream_t st, int h, int w, const float* img, const float* k25, float* out) {
    if (h < 5 || w < 5) return 0;
    if (!ring_ok(h, w, img, out)) return launch_conv5x5_f32_reg(st, h, w, img, k25, out);
    StencilArgs a = {};
    for (int t = 0; t < 25; t++) a.kf[t] = k25[t];
    a.negz = pack2(-0.0f);
    a.one = pack2(1.0f);
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h - 4 + S_BAND - 1) / S_BAND);
    stencil_ring_kernel<false, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    return (int)cudaGetLastError();
}

int launch_conv5x5_u8(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25, int* out) {
    if (h <= 0 || w <= 0) return 0;
    if (!ring_ok(h, w, img, out)) return launch_conv5x5_u8_reg(st, h, w, scale, img, k25, out);
    StencilArgs a = {};
    bool small = true;
    for (int t = 0; t < 25; t++) {
        a.kf[t] = (float)k25[t];
        a.ki[t] = k25[t];
        small &= (k25[t] >= -657 && k25[t] <= 657);  // |acc| <= 25 * 255 * 657 < 2^22
    }
    a.exact_only = small ? 0 : 1;
    a.scale = scale;
    a.shift = -1;
    if (scale > 0 && (scale & (scale - 1)) == 0) {
        a.shift = 0;
        while ((1 << a.shift) != scale) a.shift++;
    } else if (scale >= 2) {
        a.magic = ~0ull / (unsigned long long)scale + 1;
    }
    // per-device repair flag (zero between launches: the repair pass re-arms it)
    static unsigned* flags[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!flags[dev & 63]) {
        if (cudaMalloc(&flags[dev & 63], sizeof(unsigned)) != cudaSuccess) return (int)cudaErrorMemoryAllocation;
        cudaMemset(flags[dev & 63], 0, sizeof(unsigned));
    }
    a.repair_flag = flags[dev & 63];
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h + S_BAND - 1) / S_BAND);
    if (!a.exact_only) {
        if (a.shift >= 0) stencil_ring_kernel<true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else stencil_ring_kernel<true, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    }
    const long long n = (long long)h * w, blocks = (n + 255) / 256;
    u8_repair_kernel<<<(int)(blocks < PENCIL_NUM_SMS * 8 ? blocks : PENCIL_NUM_SMS * 8), 256, 0, st>>>(h, w, img, out, a);
    u8_rearm_kernel<<<1, 1, 0, st>>>(a.repair_flag);
    return (int)cudaGetLastError();
}
