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
// Rank-1 integer taps (the binomial of the bench config; any k = u (x) v with small sums) take
// the SEP kernels: rows are filtered horizontally as they enter the window and each output row
// sums 5 of them vertically — 10 FFMA2 per pixel pair instead of 25, exact in integers.
// 16384^2: int32 storage 0.413 -> 0.374 ms (88% of HBM), packed bytes 0.367 -> 0.258 ms.
// Taps supported on the radius-2 diamond (the 12 corner taps zero: sharpen, Laplacian shapes) take
// the DIA kernels, which drop the zero taps at compile time (13 instead of 25 FFMA2 per pair):
// the suite's sharpen 0.411 -> 0.364 ms on int32 storage, 0.367 -> 0.283 ms on packed bytes.
//
// Measured and dropped: two output rows per step (6-row window, four FFMA2 add chains per warp
// instead of two): 0.485 ms vs 0.475 — the f32 kernel's `wait` stalls are not chain latency;
// and a push form (each entering row added into the 5 output rows it feeds, same per-sum
// order, 80 instead of 104 registers, 6 CTAs/SM): 0.520 ms — 2.4x the MOVs.
// And a narrow f32 sweep (a lane owns one pixel pair of a 64-column strip: 5x5 window, 76
// registers, 6 CTAs/SM): 0.542 ms; 7 / 8 CTAs/SM 0.562 / 0.609 ms — more warps do not help,
// the extra per-pixel ring/loop instructions cost more than the occupancy buys.
//
// Policies (same arithmetic as the fallbacks, so the parity claims carry over unchanged):
//   F32  conv5x5_f32: interior only; acc = acc + k*img per tap in source order with the product
//        and the sum each rounded (FFMA2 against runtime -0 / 1): bit-exact vs the emitted C.
//        Taps 0 / +-2^e (e <= 0) are fused into one FFMA2 (PF kernels: k*x is exact, so one
//        rounding is the same), guarded against products below 2^-126 (f32_repair_kernel):
//        binomial/256 at 16384^2 0.475 -> 0.394 ms.
//   U8   conv5x5_u8 on int32 storage: clamp-to-edge; integer sums on the fp32 pipe (exact for
//        pixels in [0, 255] and |k| <= 657); a warp-row whose window holds a non-byte value (or
//        a launch with larger taps) takes the exact int64 path from global memory.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int S_WARPS = 4;
#ifndef STENCIL_BAND
#define STENCIL_BAND 64
#endif
constexpr int S_BAND = STENCIL_BAND;  // output rows per warp sweep of the packed-byte kernels
// ... and of the ring / band kernels, per storage (16384², tools/conv_probe.py, two rounds on one
// box): int32-storage u8 32 rows 0.355 / 0.353 ms (binomial / sharpen) against 0.364 at 64 and
// 0.372 at 128; fp32 128 rows 0.394 / 0.471 ms (PF / generic taps) against 0.396 / 0.475 at 64 and
// 0.404 / 0.487 at 32 (u8 16 rows: sharpen 0.372; fp32 256: 0.397 / 0.477); the packed-byte SWAR
// kernels are best at 64 (sharpen 0.139 vs 0.143 / 0.152 at 32 / 128).
#ifndef STENCIL_BAND_U8
#define STENCIL_BAND_U8 32
#endif
#ifndef STENCIL_BAND_F32
#define STENCIL_BAND_F32 128
#endif
template <bool U8>
__host__ __device__ constexpr int ring_band() { return U8 ? STENCIL_BAND_U8 : STENCIL_BAND_F32; }
#ifndef STENCIL_RING
#define STENCIL_RING 8
#endif
constexpr int S_RING = STENCIL_RING;  // rows per warp ring
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
__device__ __forceinline__ u64 f2fma_rm(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
// predicated cp.async (an @p guard on the instruction itself: no branch, no reconvergence)
template <int BYTES>
__device__ __forceinline__ void cp_if(bool p, void* dst, const void* src) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
        "@p cp.async.ca.shared.global [%0], [%1], %3;\n\t}" ::"r"(smem_addr(dst)),
        "l"(src), "r"((int)p), "n"(BYTES)
        : "memory");
}
template <>
__device__ __forceinline__ void cp_if<16>(bool p, void* dst, const void* src) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}" ::"r"(smem_addr(dst)),
        "l"(src), "r"((int)p)
        : "memory");
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct StencilArgs {
    float kf[25];              // taps as fp32 (exact small integers for U8)
    float ku[5], kv[5];        // U8 separable taps: k[di][dj] = ku[di] * kv[dj] (SEP kernels)
    long long ki[25];          // int taps for the exact U8 path
    u64 negz, one;             // runtime (-0, -0) and (1, 1) for the F32 exact rounding
    u64 negmag;                // runtime (-2^23, -2^23): U8 int -> float
    u64 inv_scale, half_scaled, magic2;  // U8 pow2 scale: 2^-shift, (scale/2) * 2^-shift, 1.5 * 2^23
    int scale, shift;          // U8: scale, shift >= 0 when scale = 1 << shift
    unsigned long long magic;  // U8: ceil(2^64 / scale)
    int exact_only;            // U8: taps too large for the fp32 path
    unsigned* repair_flag;     // U8: set when some window held a value outside [0, 255]
};
// The F32 kernel's arguments: StencilArgs without the separable taps.  (ptxas' register
// allocation follows the parameter layout: F32 measured 0.475 ms with this layout, 0.514 with
// ku/kv in it; the U8 kernels the other way round, 0.413 vs 0.425 ms.)
struct StencilArgsF32 {
    float kf[25];
    long long ki[25];
    u64 negz, one;
    u64 negmag;
    u64 inv_scale, half_scaled, magic2;
    int scale, shift;
    unsigned long long magic;
    int exact_only;
    unsigned* repair_flag;
    unsigned pf_lim;  // PF kernels: (|x| bits) - 1 below this marks a pixel whose scaled product may round
};

template <typename A>
__device__ __forceinline__ unsigned sat_div(long long acc, const A& a) {
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
    typedef StencilArgsF32 A;
};
template <>
struct Pol<true> {
    typedef int T;
    typedef StencilArgs A;
};

// Per-lane copy plan, fixed for the whole sweep: lane l copies columns c..c+3 (c = c0 + 4l) of
// a row to ring index 4 + 4l; lane 0 also copies the 4-column left halo (ring index 0) and lane
// 31 the right halo (ring index 132) — one extra 16-byte copy at offset `hdir` * 4.
struct RingLane {
    bool body;  // c + 3 < w
    bool halo;  // lane 0 with c0 >= 4, or lane 31 with c0 + 131 < w
    int hdir;   // -1 (left halo) or +1 (right halo)
};
__device__ __forceinline__ RingLane ring_lane(int w, int c0, int lane) {
    RingLane L;
    const int c = c0 + 4 * lane;
    L.body = c + 3 < w;
    L.halo = (lane == 0 && c0 >= 4) || (lane == 31 && c0 + 131 < w);
    L.hdir = lane == 0 ? -1 : 1;
    return L;
}
// src = &img[row][c0 + 4 * lane]
template <typename T>
__device__ __forceinline__ void ring_issue(const T* src, const RingLane& L, int lane, T* slot) {
    T* dst = slot + 4 + 4 * lane;
    if (L.body) cp16(dst, src);  // (predicated cp_if copies here measured slower for F32: 0.408 vs 0.398 ms)
    if (L.halo) cp16(dst + 4 * L.hdir, src + 4 * L.hdir);
}

// Window row entering the register window, as packed pixel-pair operands for FFMA2; e[m] =
// column c-2+m (clamped for U8).
//   F32: 7 pairs P[m] = (e[m], e[m+1]); the lane's pixel pair (c, c+1) takes tap dj from P[dj],
//        pair (c+2, c+3) from P[dj+2].  The even pairs come straight from the 8-byte-aligned
//        ring reads; the odd pairs (P[1], P[3], P[5]) share every value with an even pair, so
//        they are produced by an FFMA2 (x * 1 + -0, exact) into registers of their own — a plain
//        pack is rematerialised by ptxas at every use (~40 MOVs per output row).
//   U8:  6 pairs P[m] = (e[m], e[m+2]) for pixel pairs (c, c+2) and (c+1, c+3) (taps P[dj],
//        P[dj+1]); each pair is converted int -> float by its own LOP3s + one FFMA2, so it lands
//        in fresh registers too.  `orv` collects every value read (non-byte check).
//   F32 PF: `orv` keeps the minimum of (|x| bits) - 1 over the lane's own columns (the
//        exactness guard of the fused power-of-two taps, below).
template <bool U8, typename A, int PF = 0>
__device__ __forceinline__ void ring_read(const typename Pol<U8>::T* slot, int w, int c0, int lane,
                                          const A& a, u64 (&P)[7], unsigned& orv) {
    const int c = c0 + 4 * lane;
    // columns c-2 .. c+5 sit at ring index 4*lane+2 .. 4*lane+9: 8 B + 16 B + 8 B aligned reads
    const typename Pol<U8>::T* p = slot + 4 * lane + 2;
    u64 q[4];
    q[0] = *reinterpret_cast<const u64*>(p);
    {
        const ulonglong2 mid = *reinterpret_cast<const ulonglong2*>(p + 2);
        q[1] = mid.x;
        q[2] = mid.y;
    }
    q[3] = *reinterpret_cast<const u64*>(p + 6);
    if (U8) {
        unsigned v[8];
#pragma unroll
        for (int m = 0; m < 4; m++) {
            v[2 * m] = (unsigned)q[m];
            v[2 * m + 1] = (unsigned)(q[m] >> 32);
        }
        if (c0 == 0 || c0 + 132 > w) {  // image-edge strips: clamp-to-edge columns
#pragma unroll
            for (int m = 0; m < 8; m++) {
                const int col = c - 2 + m;
                if (col < 0 || col > w - 1) v[m] = (unsigned)slot[clampi(col, 0, w - 1) - (c0 - 4)];
            }
        }
        orv |= (v[0] | v[1] | v[2]) | (v[3] | v[4] | v[5]) | (v[6] | v[7]);
        // exact int -> float: bits (v & 255) | 0x4B000000 are 2^23 + v; the FFMA2 subtracts 2^23
#pragma unroll
        for (int m = 0; m < 6; m++) {
            const u64 bits = ((u64)((v[m + 2] & 255u) | 0x4B000000u) << 32) | ((v[m] & 255u) | 0x4B000000u);
            P[m] = f2fma(bits, a.one, a.negmag);
        }
    } else {
#pragma unroll
        for (int m = 0; m < 4; m++) P[2 * m] = q[m];
#pragma unroll
        for (int m = 0; m < 3; m++) P[2 * m + 1] = f2fma((q[m] >> 32) | (q[m + 1] << 32), a.one, a.negz);
        if (PF && c + 3 < w) {  // columns c .. c+3 (every pixel is some lane's own column)
            const unsigned x[4] = {(unsigned)q[1], (unsigned)(q[1] >> 32), (unsigned)q[2], (unsigned)(q[2] >> 32)};
#pragma unroll
            for (int t = 0; t < 4; t++) orv = min(orv, (x[t] & 0x7fffffffu) - 1u);
        }
    }
}

// A row entering the window.  Full 5x5 taps: the row's operand pairs as they are.  SEP
// (integer taps of rank 1, k = ku (x) kv): the row is filtered horizontally on entry — pairs
// (c, c+2) and (c+1, c+3) of sum_dj kv[dj] * e[m+dj] — so each output row then costs 5
// vertical FFMA2 per pair instead of 25.  Integer sums regroup exactly (all partial sums stay
// below 2^22), so the result is the full 25-tap sum bit for bit.
template <bool SEP, typename A>
__device__ __forceinline__ void enter_row(const u64 (&P)[7], u64 (&Wr)[7], const A& a) {
    if constexpr (SEP) {
        u64 h02 = 0ull, h13 = 0ull;
#pragma unroll
        for (int dj = 0; dj < 5; dj++) {
            const u64 kk = f2pk(a.kv[dj], a.kv[dj]);
            h02 = f2fma(kk, P[dj], h02);
            h13 = f2fma(kk, P[dj + 1], h13);
        }
        Wr[0] = h02;
        Wr[1] = h13;
    } else {
#pragma unroll
        for (int m = 0; m < 7; m++) Wr[m] = P[m];
    }
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

// Row band of a band-sharded image (multi-GPU row bands, halo rows read in place): the two rows
// above the band and the two below, as row pointers — the neighbour ranks' edge rows through
// their NVLink peer mappings, or the band's own edge row repeated at the image's top / bottom
// (clamp-to-edge).  out_lo / out_hi: the band-relative output rows (f32: the image interior).
template <typename T>
struct BandSrc {
    const T* top[2];  // rows -2, -1
    const T* bot[2];  // rows h, h + 1
    int out_lo, out_hi;
};

// Sweep state advanced by one row per step: `src` points at the lane's columns of the next row
// to enter the ring (rows past the image bottom clamp to `src_last` for U8), `dst` at the
// lane's columns of the output row.
template <typename T>
struct Sweep {
    const T* src;
    const T* src_last;
    T* dst;
    long long w;
};

// F32 taps fused into one FFMA2 by the PF kernels: PF 1 = the 16 taps off the centre row and
// column (the binomial's powers of two), PF 2 = all 25.
__host__ __device__ constexpr bool pf_tap(int pf, int di, int dj) {
    return pf == 2 || (pf == 1 && di != 2 && dj != 2);
}

template <bool U8, int S, bool POW2, bool SEP, bool BAND = false, bool DIA = false, int PF = 0>
__device__ __forceinline__ void stencil_step(int w, int i, int c, int lane, int r_end, const RingLane& L,
                                             typename Pol<U8>::T (*ring)[S_ROWE], u64 (&W)[5][7],
                                             Sweep<typename Pol<U8>::T>& sw, unsigned& orv,
                                             const typename Pol<U8>::A& a,
                                             const BandSrc<typename Pol<U8>::T>* bs = nullptr, int h = 0) {
    typedef typename Pol<U8>::T T;
    // the ring holds rows i+2 .. i+2+S_RING-1 in flight; the oldest (row i+2) must have landed
    cp_wait<S_RING - 1>();
    __syncwarp();
    T* slot = ring[(i + 2) % S_RING];
    {
        u64 P[7];
        ring_read<U8, typename Pol<U8>::A, PF>(slot, w, c - 4 * lane, lane, a, P, orv);
        enter_row<SEP>(P, W[S], a);
    }
    __syncwarp();
    if (i + 2 + S_RING < r_end) {
        const T* src = sw.src;
        if constexpr (BAND) {  // rows h, h + 1: the lower halo
            const int r = i + 2 + S_RING;
            if (r >= h) src = (r == h ? bs->bot[0] : bs->bot[1]) + c;
        } else if (U8 && src > sw.src_last) {
            src = sw.src_last;  // clamp-to-edge rows below the image
        }
        ring_issue<T>(src, L, lane, slot);
    }
    cp_commit();
    sw.src += sw.w;

    u64 a01 = 0ull, a23 = 0ull;  // pixel pairs (c, c+1) and (c+2, c+3)
#pragma unroll
    for (int di = 0; di < 5; di++) {
        const int sl = (S + 1 + di) % 5;
        if constexpr (SEP) {  // vertical pass over the horizontally filtered rows
            const u64 kk = f2pk(a.ku[di], a.ku[di]);
            a01 = f2fma(kk, W[sl][0], a01);
            a23 = f2fma(kk, W[sl][1], a23);
            continue;
        }
#pragma unroll
        for (int dj = 0; dj < 5; dj++) {
            if (DIA && (di - 2 < 0 ? 2 - di : di - 2) + (dj - 2 < 0 ? 2 - dj : dj - 2) > 2) continue;  // zero tap
            const u64 kk = f2pk(a.kf[di * 5 + dj], a.kf[di * 5 + dj]);
            if (U8) {  // exact integer sums: fused is fine
                a01 = f2fma(kk, W[sl][dj], a01);      // pixels (c, c+2)
                a23 = f2fma(kk, W[sl][dj + 1], a23);  // pixels (c+1, c+3)
            } else if (pf_tap(PF, di, dj)) {  // k = 0 or +-2^e: k*x is exact, so one rounding is the same
                a01 = f2fma(kk, W[sl][dj], a01);
                a23 = f2fma(kk, W[sl][dj + 2], a23);
            } else {   // product and sum rounded separately, as written (runtime -0 / 1: with
                       // mul.rn.f32x2 + add.rn.f32x2 ptxas emits one fused FFMA2 — wrong results)
                a01 = f2fma(f2fma(kk, W[sl][dj], a.negz), a.one, a01);
                a23 = f2fma(f2fma(kk, W[sl][dj + 2], a.negz), a.one, a23);
            }
        }
    }
    T* orow = sw.dst;
    sw.dst += sw.w;
    if (U8) {
        int v[4];
        if (POW2) {
            // (acc + scale/2) >> shift on the pair: t = (acc + scale/2) * 2^-shift is exact, and
            // t + 1.5 * 2^23 rounded toward -inf holds floor(t) in its low mantissa bits
            const float2 f02 = f2unpk(f2fma_rm(f2fma(a01, a.inv_scale, a.half_scaled), a.one, a.magic2));
            const float2 f13 = f2unpk(f2fma_rm(f2fma(a23, a.inv_scale, a.half_scaled), a.one, a.magic2));
            const float f[4] = {f02.x, f13.x, f02.y, f13.y};
#pragma unroll
            for (int t = 0; t < 4; t++) v[t] = __vimin_s32_relu(__float_as_int(f[t]) - 0x4B400000, 255);
        } else {
            const float2 p02 = f2unpk(a01), p13 = f2unpk(a23);
            const float o[4] = {p02.x, p13.x, p02.y, p13.y};
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int acc = __float_as_int(__fadd_rn(o[t], 12582912.f)) - 0x4B400000;  // exact, |acc| < 2^22
                v[t] = (int)sat_div(acc, a);
            }
        }
        if (L.body) *reinterpret_cast<int4*>((int*)orow) = make_int4(v[0], v[1], v[2], v[3]);
    } else {
        const float2 p01 = f2unpk(a01), p23 = f2unpk(a23);
        const float o[4] = {p01.x, p01.y, p23.x, p23.y};
        if (c >= 2 && c + 3 < w - 2) {
            st_stream_f4(reinterpret_cast<float4*>((float*)orow), make_float4(o[0], o[1], o[2], o[3]));
        } else {
#pragma unroll
            for (int t = 0; t < 4; t++)
                if (c + t >= 2 && c + t < w - 2) ((float*)orow)[t] = o[t];
        }
    }
}

#ifndef STENCIL_F32_MINB
#define STENCIL_F32_MINB 4
#endif
#ifndef STENCIL_U8_MINB
#define STENCIL_U8_MINB 4
#endif
#ifndef STENCIL_SEP_MINB  // swept 4/5/6/8 at 16384^2: int32 0.374/0.374/0.376/0.378 ms, bytes 0.258/0.258/0.262/0.279;
                          // again at 32-row bands (round 2): 4/5/6 0.355/0.355/0.361 ms
#define STENCIL_SEP_MINB 4
#endif
template <bool U8, bool POW2, bool SEP = false, bool DIA = false, int PF = 0>
__global__ void __launch_bounds__(32 * S_WARPS, SEP ? STENCIL_SEP_MINB : (U8 ? STENCIL_U8_MINB : STENCIL_F32_MINB)) stencil_ring_kernel(
    int h, int w, const typename Pol<U8>::T* __restrict__ img, typename Pol<U8>::T* __restrict__ out,
    typename Pol<U8>::A a) {
    typedef typename Pol<U8>::T T;
    __shared__ __align__(16) T ring_all[S_WARPS][S_RING][S_ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int strip = blockIdx.x * S_WARPS + warp;
    const int c0 = strip * 128;
    if (c0 >= w) return;
    const int c = c0 + 4 * lane;
    // output rows [i0, i1); input rows [i0 - 2, i1 + 2)
    const int i0 = (U8 ? 0 : 2) + blockIdx.y * ring_band<U8>();
    const int i1 = min(U8 ? h : h - 2, i0 + ring_band<U8>());
    if (i0 >= i1) return;
    const int r_end = i1 + 2;
    const RingLane L = ring_lane(w, c0, lane);
    T(*ring)[S_ROWE] = ring_all[warp];
    auto row_src = [&](int r) { return img + (long long)(U8 ? clampi(r, 0, h - 1) : r) * w + c; };
#pragma unroll
    for (int d = 0; d < S_RING; d++) {  // prologue: rows i0-2 .. i0+5 in flight
        if (i0 - 2 + d < r_end) ring_issue<T>(row_src(i0 - 2 + d), L, lane, ring[(i0 - 2 + d + S_RING) % S_RING]);
        cp_commit();
    }
    u64 W[5][7];
    unsigned orv = PF ? ~0u : 0u;
#pragma unroll
    for (int d = 0; d < 4; d++) {  // rows i0-2 .. i0+1 into the window, slots refilled
        cp_wait<S_RING - 1>();
        __syncwarp();
        T* slot = ring[(i0 - 2 + d + S_RING) % S_RING];
        {
            u64 P[7];
            ring_read<U8, typename Pol<U8>::A, PF>(slot, w, c0, lane, a, P, orv);
            enter_row<SEP>(P, W[d], a);
        }
        __syncwarp();
        if (i0 - 2 + d + S_RING < r_end) ring_issue<T>(row_src(i0 - 2 + d + S_RING), L, lane, slot);
        cp_commit();
    }
    Sweep<T> sw;
    sw.w = w;
    sw.src_last = img + (long long)(h - 1) * w + c;
    sw.src = img + (long long)(i0 + 2 + S_RING) * w + c;  // next row to enter the ring: i0 + 2 + S_RING
    sw.dst = out + (long long)i0 * w + c;
    for (int i = i0; i < i1; i += 5) {
        stencil_step<U8, 4, POW2, SEP, false, DIA, PF>(w, i, c, lane, r_end, L, ring, W, sw, orv, a);
        if (i + 1 < i1) stencil_step<U8, 0, POW2, SEP, false, DIA, PF>(w, i + 1, c, lane, r_end, L, ring, W, sw, orv, a);
        if (i + 2 < i1) stencil_step<U8, 1, POW2, SEP, false, DIA, PF>(w, i + 2, c, lane, r_end, L, ring, W, sw, orv, a);
        if (i + 3 < i1) stencil_step<U8, 2, POW2, SEP, false, DIA, PF>(w, i + 3, c, lane, r_end, L, ring, W, sw, orv, a);
        if (i + 4 < i1) stencil_step<U8, 3, POW2, SEP, false, DIA, PF>(w, i + 4, c, lane, r_end, L, ring, W, sw, orv, a);
    }
    cp_wait<0>();
    // a non-byte pixel anywhere in the sweep: flag the launch for the exact repair pass
    // (u8_repair_kernel), which recomputes the whole image in int64
    if (U8 && __any_sync(0xffffffffu, (orv & ~255u) != 0) && lane == 0) atomicOr(a.repair_flag, 1u);
    // PF: a pixel with 0 < |x| < 2^(-126 - emin) (a fused tap's product could round in the
    // subnormal range): flag the launch for f32_repair_kernel
    if constexpr (!U8 && PF != 0)
        if (__any_sync(0xffffffffu, orv < a.pf_lim) && lane == 0) atomicOr(a.repair_flag, 1u);
}

// Exact pass behind the PF kernels: exits at once unless the fast kernel flagged a pixel outside
// the fused taps' exact range; then recomputes every interior pixel as written (product and sum
// rounded separately, source order).  The last CTA out re-arms the flag (flag[1] counts CTAs),
// so the common case costs one near-empty launch.
__global__ void f32_repair_kernel(int h, int w, const float* __restrict__ img, float* __restrict__ out,
                                  StencilArgsF32 a) {
    if (*(volatile unsigned*)a.repair_flag == 0) return;
    const long long iw = w - 4, n = (long long)(h - 4) * iw;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const long long i = 2 + p / iw, j = 2 + p % iw;
        float acc = 0.f;
#pragma unroll 1
        for (int di = 0; di < 5; di++)
#pragma unroll
            for (int dj = 0; dj < 5; dj++)
                acc = __fadd_rn(acc, __fmul_rn(a.kf[di * 5 + dj], img[(i + di - 2) * w + j + dj - 2]));
        out[i * w + j] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.repair_flag + 1, 1u) == gridDim.x - 1) {
            a.repair_flag[1] = 0u;
            *(volatile unsigned*)a.repair_flag = 0u;
        }
    }
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

// ---------------------------------------------------------------- band-sharded sweep
// One rank's row band of a band-sharded image with the halo exchange fused away: the rows above
// and below the band are read where they live (BandSrc: the neighbours' edge rows through NVLink
// peer mappings, cp.async straight into the ring), so a multi-GPU stencil step is one launch per
// rank and no halo copy.  Same sweep, arithmetic and policies as stencil_ring_kernel (the output
// is bit-identical to the single-GPU image's rows); h = the band's own rows.
template <bool U8, bool POW2, bool SEP = false, bool DIA = false, int PF = 0>
__global__ void __launch_bounds__(32 * S_WARPS, SEP ? STENCIL_SEP_MINB : (U8 ? STENCIL_U8_MINB : STENCIL_F32_MINB)) stencil_band_kernel(
    int h, int w, const typename Pol<U8>::T* __restrict__ img, typename Pol<U8>::T* __restrict__ out,
    typename Pol<U8>::A a, BandSrc<typename Pol<U8>::T> bs) {
    typedef typename Pol<U8>::T T;
    __shared__ __align__(16) T ring_all[S_WARPS][S_RING][S_ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = (blockIdx.x * S_WARPS + warp) * 128;
    if (c0 >= w) return;
    const int c = c0 + 4 * lane;
    const int i0 = bs.out_lo + blockIdx.y * ring_band<U8>();
    const int i1 = min(bs.out_hi, i0 + ring_band<U8>());
    if (i0 >= i1) return;
    const int r_end = i1 + 2;
    const RingLane L = ring_lane(w, c0, lane);
    T(*ring)[S_ROWE] = ring_all[warp];
    auto row_src = [&](int r) {
        return (r < 0 ? (r == -2 ? bs.top[0] : bs.top[1]) : (r >= h ? (r == h ? bs.bot[0] : bs.bot[1]) : img + (long long)r * w)) + c;
    };
#pragma unroll
    for (int d = 0; d < S_RING; d++) {  // prologue: rows i0-2 .. i0+5 in flight
        if (i0 - 2 + d < r_end) ring_issue<T>(row_src(i0 - 2 + d), L, lane, ring[(i0 - 2 + d + S_RING) % S_RING]);
        cp_commit();
    }
    u64 W[5][7];
    unsigned orv = PF ? ~0u : 0u;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        cp_wait<S_RING - 1>();
        __syncwarp();
        T* slot = ring[(i0 - 2 + d + S_RING) % S_RING];
        {
            u64 P[7];
            ring_read<U8, typename Pol<U8>::A, PF>(slot, w, c0, lane, a, P, orv);
            enter_row<SEP>(P, W[d], a);
        }
        __syncwarp();
        if (i0 - 2 + d + S_RING < r_end) ring_issue<T>(row_src(i0 - 2 + d + S_RING), L, lane, slot);
        cp_commit();
    }
    Sweep<T> sw;
    sw.w = w;
    sw.src_last = nullptr;
    sw.src = img + (long long)(i0 + 2 + S_RING) * w + c;
    sw.dst = out + (long long)i0 * w + c;
    for (int i = i0; i < i1; i += 5) {
        stencil_step<U8, 4, POW2, SEP, true, DIA, PF>(w, i, c, lane, r_end, L, ring, W, sw, orv, a, &bs, h);
        if (i + 1 < i1) stencil_step<U8, 0, POW2, SEP, true, DIA, PF>(w, i + 1, c, lane, r_end, L, ring, W, sw, orv, a, &bs, h);
        if (i + 2 < i1) stencil_step<U8, 1, POW2, SEP, true, DIA, PF>(w, i + 2, c, lane, r_end, L, ring, W, sw, orv, a, &bs, h);
        if (i + 3 < i1) stencil_step<U8, 2, POW2, SEP, true, DIA, PF>(w, i + 3, c, lane, r_end, L, ring, W, sw, orv, a, &bs, h);
        if (i + 4 < i1) stencil_step<U8, 3, POW2, SEP, true, DIA, PF>(w, i + 4, c, lane, r_end, L, ring, W, sw, orv, a, &bs, h);
    }
    cp_wait<0>();
    if (U8 && __any_sync(0xffffffffu, (orv & ~255u) != 0) && lane == 0) atomicOr(a.repair_flag, 1u);
    if constexpr (!U8 && PF != 0)  // as stencil_ring_kernel: a pixel the fused taps cannot take exactly
        if (__any_sync(0xffffffffu, orv < a.pf_lim) && lane == 0) atomicOr(a.repair_flag, 1u);
}

// f32_repair_kernel for a band: the band's output rows [out_lo, out_hi) as written, the halo rows
// read where they live (BandSrc); exits at once unless the PF band sweep flagged a pixel
__global__ void f32_band_repair_kernel(int h, int w, const float* __restrict__ img, float* __restrict__ out,
                                       StencilArgsF32 a, BandSrc<float> bs) {
    if (*(volatile unsigned*)a.repair_flag == 0) return;
    const long long iw = w - 4, n = (long long)(bs.out_hi - bs.out_lo) * iw;
    auto row = [&](int r) -> const float* {
        return r < 0 ? (r == -2 ? bs.top[0] : bs.top[1]) : (r >= h ? (r == h ? bs.bot[0] : bs.bot[1]) : img + (long long)r * w);
    };
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const int i = bs.out_lo + (int)(p / iw), j = 2 + (int)(p % iw);
        float acc = 0.f;
#pragma unroll 1
        for (int di = 0; di < 5; di++) {
            const float* rp = row(i + di - 2);
#pragma unroll
            for (int dj = 0; dj < 5; dj++) acc = __fadd_rn(acc, __fmul_rn(a.kf[di * 5 + dj], rp[j + dj - 2]));
        }
        out[(long long)i * w + j] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.repair_flag + 1, 1u) == gridDim.x - 1) {
            a.repair_flag[1] = 0u;
            *(volatile unsigned*)a.repair_flag = 0u;
        }
    }
}

// the exact int64 repair pass of a band (rows outside it through BandSrc)
__global__ void u8_band_repair_kernel(int h, int w, const int* __restrict__ img, int* __restrict__ out,
                                      StencilArgs a, BandSrc<int> bs) {
    if (!a.exact_only && *(volatile unsigned*)a.repair_flag == 0) return;
    const long long n = (long long)h * w;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(p / w), j = (int)(p % w);
        long long acc = 0;
#pragma unroll 1
        for (int di = 0; di < 5; di++) {
            const int r = i + di - 2;
            const int* row = r < 0 ? (r == -2 ? bs.top[0] : bs.top[1]) : (r >= h ? (r == h ? bs.bot[0] : bs.bot[1]) : img + (long long)r * w);
#pragma unroll 1
            for (int dj = 0; dj < 5; dj++) acc += a.ki[di * 5 + dj] * (long long)row[clampi(j + dj - 2, 0, w - 1)];
        }
        out[p] = (int)sat_div(acc, a);
    }
}

// ---------------------------------------------------------------- packed 8-bit images
// conv5x5_u8 semantics on 1-byte pixels (pencil_conv5x5_u8_bytes_dev): the same sweep with a
// byte ring (136 bytes per row: columns [c0 - 4, c0 + 132)), filled by 4-byte cp.async per
// lane.  A lane owns 4 pixels; its 8 window bytes come from 3 ring words, each pixel pair is
// built by two PRMTs (byte | 0x4B000000 = 2^23 + v) and one FFMA2 (- 2^23), then the same
// 25 fused FFMA2 per pair and pairwise requantisation as the int32-storage kernel; the 4 output
// bytes leave as one 32-bit store.  Taps are limited to |k| <= 657 (exact fp32 sums); larger
// taps take the dp4a / scalar kernels of k_conv_u8b.cu.
constexpr int SB_ROWE = 136;

__device__ __forceinline__ void cp4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ u64 byte_pair(unsigned wlo, int blo, unsigned whi, int bhi, const StencilArgs& a) {
    const unsigned lo = __byte_perm(wlo, 0x4B000000u, 0x7540u + blo);
    const unsigned hi = __byte_perm(whi, 0x4B000000u, 0x7540u + bhi);
    return f2fma(((u64)hi << 32) | lo, a.one, a.negmag);
}

// window row of the lane (columns c-2 .. c+5) as pairs P[m] = (e[m], e[m+2]), m = 0..5
__device__ __forceinline__ void bytes_read(const unsigned char* slot, int w, int c0, int lane, const StencilArgs& a,
                                           u64 (&P)[7]) {
    const unsigned* wp = reinterpret_cast<const unsigned*>(slot) + lane;  // ring words lane .. lane+2
    unsigned W0 = wp[0], W1 = wp[1], W2 = wp[2];  // columns c-4..c-1 | c..c+3 | c+4..c+7
    const int c = c0 + 4 * lane;
    if (c0 == 0 || c0 + 132 > w) {  // image-edge strips: clamp-to-edge columns
        unsigned char v[8];
#pragma unroll
        for (int m = 0; m < 8; m++) {
            const int col = c - 2 + m;
            v[m] = slot[clampi(col, 0, w - 1) - (c0 - 4)];
        }
        W0 = ((unsigned)v[0] << 16) | ((unsigned)v[1] << 24);
        W1 = v[2] | ((unsigned)v[3] << 8) | ((unsigned)v[4] << 16) | ((unsigned)v[5] << 24);
        W2 = v[6] | ((unsigned)v[7] << 8);
    }
    // e[m] = byte (m + 2) of the 12-byte run W0 W1 W2
    P[0] = byte_pair(W0, 2, W1, 0, a);
    P[1] = byte_pair(W0, 3, W1, 1, a);
    P[2] = byte_pair(W1, 0, W1, 2, a);
    P[3] = byte_pair(W1, 1, W1, 3, a);
    P[4] = byte_pair(W1, 2, W2, 0, a);
    P[5] = byte_pair(W1, 3, W2, 1, a);
}

template <int S, bool POW2, bool SEP, bool DIA = false>
__device__ __forceinline__ void bytes_step(int w, int i, int c, int lane, int r_end, const RingLane& L,
                                           unsigned char (*ring)[SB_ROWE], u64 (&W)[5][7],
                                           Sweep<unsigned char>& sw, const StencilArgs& a) {
    cp_wait<S_RING - 1>();
    __syncwarp();
    unsigned char* slot = ring[(i + 2) % S_RING];
    {
        u64 P[7];
        bytes_read(slot, w, c - 4 * lane, lane, a, P);
        enter_row<SEP>(P, W[S], a);
    }
    __syncwarp();
    if (i + 2 + S_RING < r_end) {
        const unsigned char* src = sw.src > sw.src_last ? sw.src_last : sw.src;
        unsigned char* dst = slot + 4 + 4 * lane;
        if (L.body) cp4(dst, src);
        if (L.halo) cp4(dst + 4 * L.hdir, src + 4 * L.hdir);
    }
    cp_commit();
    sw.src += sw.w;
    u64 a02 = 0ull, a13 = 0ull;
#pragma unroll
    for (int di = 0; di < 5; di++) {
        const int sl = (S + 1 + di) % 5;
        if constexpr (SEP) {
            const u64 kk = f2pk(a.ku[di], a.ku[di]);
            a02 = f2fma(kk, W[sl][0], a02);
            a13 = f2fma(kk, W[sl][1], a13);
            continue;
        }
#pragma unroll
        for (int dj = 0; dj < 5; dj++) {
            if (DIA && (di - 2 < 0 ? 2 - di : di - 2) + (dj - 2 < 0 ? 2 - dj : dj - 2) > 2) continue;  // zero tap
            const u64 kk = f2pk(a.kf[di * 5 + dj], a.kf[di * 5 + dj]);
            a02 = f2fma(kk, W[sl][dj], a02);
            a13 = f2fma(kk, W[sl][dj + 1], a13);
        }
    }
    unsigned char* orow = sw.dst;
    sw.dst += sw.w;
    int v[4];
    if (POW2) {
        const float2 f02 = f2unpk(f2fma_rm(f2fma(a02, a.inv_scale, a.half_scaled), a.one, a.magic2));
        const float2 f13 = f2unpk(f2fma_rm(f2fma(a13, a.inv_scale, a.half_scaled), a.one, a.magic2));
        const float f[4] = {f02.x, f13.x, f02.y, f13.y};
#pragma unroll
        for (int t = 0; t < 4; t++) v[t] = __vimin_s32_relu(__float_as_int(f[t]) - 0x4B400000, 255);
    } else {
        const float2 p02 = f2unpk(a02), p13 = f2unpk(a13);
        const float o[4] = {p02.x, p13.x, p02.y, p13.y};
#pragma unroll
        for (int t = 0; t < 4; t++)
            v[t] = (int)sat_div(__float_as_int(__fadd_rn(o[t], 12582912.f)) - 0x4B400000, a);
    }
    if (L.body)
        *reinterpret_cast<unsigned*>(orow) =
            (unsigned)v[0] | ((unsigned)v[1] << 8) | ((unsigned)v[2] << 16) | ((unsigned)v[3] << 24);
}

template <bool POW2, bool SEP = false, bool DIA = false>
__global__ void __launch_bounds__(32 * S_WARPS, SEP ? STENCIL_SEP_MINB : STENCIL_U8_MINB) stencil_bytes_kernel(int h, int w,
                                                                                 const unsigned char* __restrict__ img,
                                                                                 unsigned char* __restrict__ out,
                                                                                 StencilArgs a) {
    __shared__ __align__(16) unsigned char ring_all[S_WARPS][S_RING][SB_ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = (blockIdx.x * S_WARPS + warp) * 128;
    if (c0 >= w) return;
    const int c = c0 + 4 * lane;
    const int i0 = blockIdx.y * S_BAND, i1 = min(h, i0 + S_BAND);
    if (i0 >= i1) return;
    const int r_end = i1 + 2;
    const RingLane L = ring_lane(w, c0, lane);
    unsigned char(*ring)[SB_ROWE] = ring_all[warp];
    auto issue = [&](int r, unsigned char* slot) {
        const unsigned char* src = img + (long long)clampi(r, 0, h - 1) * w + c;
        unsigned char* dst = slot + 4 + 4 * lane;
        if (L.body) cp4(dst, src);
        if (L.halo) cp4(dst + 4 * L.hdir, src + 4 * L.hdir);
    };
#pragma unroll
    for (int d = 0; d < S_RING; d++) {
        if (i0 - 2 + d < r_end) issue(i0 - 2 + d, ring[(i0 - 2 + d + S_RING) % S_RING]);
        cp_commit();
    }
    u64 W[5][7];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        cp_wait<S_RING - 1>();
        __syncwarp();
        unsigned char* slot = ring[(i0 - 2 + d + S_RING) % S_RING];
        {
            u64 P[7];
            bytes_read(slot, w, c0, lane, a, P);
            enter_row<SEP>(P, W[d], a);
        }
        __syncwarp();
        if (i0 - 2 + d + S_RING < r_end) issue(i0 - 2 + d + S_RING, slot);
        cp_commit();
    }
    Sweep<unsigned char> sw;
    sw.w = w;
    sw.src_last = img + (long long)(h - 1) * w + c;
    sw.src = img + (long long)(i0 + 2 + S_RING) * w + c;
    sw.dst = out + (long long)i0 * w + c;
    for (int i = i0; i < i1; i += 5) {
        bytes_step<4, POW2, SEP, DIA>(w, i, c, lane, r_end, L, ring, W, sw, a);
        if (i + 1 < i1) bytes_step<0, POW2, SEP, DIA>(w, i + 1, c, lane, r_end, L, ring, W, sw, a);
        if (i + 2 < i1) bytes_step<1, POW2, SEP, DIA>(w, i + 2, c, lane, r_end, L, ring, W, sw, a);
        if (i + 3 < i1) bytes_step<2, POW2, SEP, DIA>(w, i + 3, c, lane, r_end, L, ring, W, sw, a);
        if (i + 4 < i1) bytes_step<3, POW2, SEP, DIA>(w, i + 4, c, lane, r_end, L, ring, W, sw, a);
    }
    cp_wait<0>();
}

u64 pack2(float v) {
    unsigned u;
    memcpy(&u, &v, 4);
    return ((u64)u << 32) | u;
}

// Integer rank-1 factorisation k = u (x) v (v primitive), or false.  Taken only when every
// partial sum of the separable order stays exact on the fp32 pipe: 255 * sum|u| * sum|v| < 2^22.
bool separable(const int* k, StencilArgs& a) {
    int r = -1;
    for (int i = 0; i < 5 && r < 0; i++)
        for (int j = 0; j < 5; j++)
            if (k[i * 5 + j]) { r = i; break; }
    if (r < 0) return false;  // all-zero taps: the general kernel
    long long g = 0;
    for (int j = 0; j < 5; j++) {
        long long x = k[r * 5 + j] < 0 ? -(long long)k[r * 5 + j] : k[r * 5 + j];
        while (x) { long long t = g % x; g = x; x = t; }
    }
    long long v[5], u[5], su = 0, sv = 0;
    int j0 = 0;
    for (int j = 0; j < 5; j++) {
        v[j] = k[r * 5 + j] / g;
        if (v[j] && !v[j0]) j0 = j;
        sv += v[j] < 0 ? -v[j] : v[j];
    }
    for (int i = 0; i < 5; i++) {
        if (k[i * 5 + j0] % v[j0]) return false;
        u[i] = k[i * 5 + j0] / v[j0];
        for (int j = 0; j < 5; j++)
            if ((long long)k[i * 5 + j] != u[i] * v[j]) return false;
        su += u[i] < 0 ? -u[i] : u[i];
    }
    if (255ll * su * sv >= (1ll << 22)) return false;
    for (int t = 0; t < 5; t++) {
        a.ku[t] = (float)u[t];
        a.kv[t] = (float)v[t];
    }
    return true;
}


// ---------------------------------------------------------------- SWAR packed-byte sweep
// Rank-1 taps k = u (x) v with u, v >= 0, a power-of-two scale and every sum below 2^16
// (255 * sum u * sum v + scale/2 < 65536, result <= 255 without a clamp: the binomial/256 of the
// config): the sums run as two 16-bit lanes per 32-bit register (SWAR) on the integer pipes
// instead of as fp32 pairs.  Unpacking is a funnel shift + one PRMT per byte pair (no int->float),
// each tap one IMAD on two pixels, requantisation one IADD + one PRMT per 4 pixels (scale 256) —
// and since a pixel pair costs one register instead of two, a lane owns 16 pixels (512-column
// strips; 8 when w % 16 != 0), quartering the per-row ring / sync / pointer overhead per pixel
// (16384^2 binomial/256: fp32-pair kernel 0.258 ms, NP 8 0.142 ms, NP 16 0.128 ms).  Integer sums: exact,
// bit-identical to the other kernels.
// NP pixels per lane (8 or 16): 32*NP-column strips; ring row = [pad | body | pad], pad = NP bytes
// (16-byte-aligned bodies for 16-byte cp.async), left halo at pad-4, right halo after the body.
template <int NP>
struct SwarGeom {
    static constexpr int PAD = NP, ROWE = 2 * NP + 32 * NP, NW = NP / 4;
};

struct SwarArgs {
    unsigned u[5], v[5];  // vertical / horizontal taps (non-negative)
    unsigned half2;       // (scale / 2) in both 16-bit lanes
    int shift;            // log2(scale) <= 8
};

__device__ __forceinline__ void cp8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
template <int NP>
__device__ __forceinline__ void cp_body(void* dst, const void* src) {
    if constexpr (NP == 16) cp16(dst, src);
    else cp8(dst, src);
}

// The row entering the window as byte pairs: Q[m] = (e[c-2+m], e[c+m]) in 16-bit lanes
// (m = 0..NP+1); output pair t (pixels c+b, c+b+2 with b = (t & 1) + 4 (t >> 1)) has its centre
// pair at Q[b + 2].  The lane's 16 body bytes are one 128-bit shared load, its two 4-byte
// neighbours two 32-bit loads.
template <int NP, bool EDGE>
__device__ __forceinline__ void swar_pairs(const unsigned char* slot, int w, int c0, int lane,
                                             unsigned (&Q)[NP + 2]) {
    typedef SwarGeom<NP> G;
    const unsigned char* body = slot + G::PAD + NP * lane;
    unsigned Wd[G::NW + 2];
    Wd[0] = *reinterpret_cast<const unsigned*>(body - 4);
    if constexpr (NP == 16) {
        const uint4 v = *reinterpret_cast<const uint4*>(body);
        Wd[1] = v.x, Wd[2] = v.y, Wd[3] = v.z, Wd[4] = v.w;
    } else {
        const uint2 v = *reinterpret_cast<const uint2*>(body);
        Wd[1] = v.x, Wd[2] = v.y;
    }
    Wd[G::NW + 1] = *reinterpret_cast<const unsigned*>(body + NP);
    if (EDGE && (c0 == 0 || c0 + 32 * NP >= w)) {  // image-edge strips: clamp-to-edge columns
        const int c = c0 + NP * lane;
        unsigned v[NP + 4];
#pragma unroll
        for (int m = 0; m < NP + 4; m++) v[m] = slot[clampi(c - 2 + m, 0, w - 1) - (c0 - G::PAD)];
        Wd[0] = (v[0] << 16) | (v[1] << 24);
#pragma unroll
        for (int k = 0; k < G::NW; k++)
            Wd[k + 1] = v[4 * k + 2] | (v[4 * k + 3] << 8) | (v[4 * k + 4] << 16) | (v[4 * k + 5] << 24);
        Wd[G::NW + 1] = v[NP + 2] | (v[NP + 3] << 8);
    }
#pragma unroll
    for (int k = 0; k <= 2 * G::NW; k++) {
        const unsigned X = (k & 1) ? Wd[k / 2 + 1] : __funnelshift_r(Wd[k / 2], Wd[k / 2 + 1], 16);
        Q[2 * k] = __byte_perm(X, 0u, 0x4240);
        Q[2 * k + 1] = __byte_perm(X, 0u, 0x4341);
    }
}

// predicated 8- / 16-byte row store (no branch around it)
template <int NP>
__device__ __forceinline__ void swar_store_if(bool p, unsigned char* dst, const unsigned (&r)[NP / 4]) {
    if constexpr (NP == 16)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %0, 0;\n\t@p st.global.v4.b32 [%1], {%2, %3, %4, %5};\n\t}"
                     ::"r"((int)p), "l"(dst), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %0, 0;\n\t@p st.global.v2.b32 [%1], {%2, %3};\n\t}"
                     ::"r"((int)p), "l"(dst), "r"(r[0]), "r"(r[1]) : "memory");
}

// Row entering the window, filtered horizontally: H[t] = u16x2 pixel pairs; t = 2g + p holds
// (c + 4g + p, c + 4g + p + 2).  SYM (v mirror-symmetric): v0 (Q[b] + Q[b+4]) + v1 (Q[b+1] + Q[b+3])
// + v2 Q[b+2], 3 IMADs + 2 adds instead of 5 IMADs (exact: the word arithmetic is linear mod 2^32
// and every final lane lies in [0, 2^16)).
template <int NP, bool SYM>
__device__ __forceinline__ void swar_enter(const unsigned char* slot, int w, int c0, int lane, const SwarArgs& a,
                                           unsigned (&H)[NP / 2]) {
    unsigned Q[NP + 2];
    swar_pairs<NP, true>(slot, w, c0, lane, Q);
#pragma unroll
    for (int t = 0; t < NP / 2; t++) {
        const int b = (t & 1) + 4 * (t >> 1);
        if (SYM) {
            H[t] = a.v[0] * (Q[b] + Q[b + 4]) + a.v[1] * (Q[b + 1] + Q[b + 3]) + a.v[2] * Q[b + 2];
        } else {
            unsigned acc = a.v[0] * Q[b];
#pragma unroll
            for (int dj = 1; dj < 5; dj++) acc += a.v[dj] * Q[b + dj];
            H[t] = acc;
        }
    }
}

// the lane's NP body bytes, and for lanes 0 / 31 of inner strips the 4 halo bytes beyond them
template <int NP>
__device__ __forceinline__ void swar_issue(const unsigned char* src, unsigned char* slot, int lane, bool body,
                                           bool halo) {
    unsigned char* dst = slot + SwarGeom<NP>::PAD + NP * lane;
    cp_if<NP>(body, dst, src);
    const int hd = lane == 0 ? -4 : NP;
    cp_if<4>(halo, dst + hd, src + hd);
}

template <int NP, int S, bool SH8, bool SYM>
__device__ __forceinline__ void swar_step(int w, int i, int c, int lane, int r_end, bool body, bool halo,
                                          unsigned char (*ring)[SwarGeom<NP>::ROWE], unsigned (&H)[5][NP / 2],
                                          Sweep<unsigned char>& sw, const SwarArgs& a) {
    cp_wait<S_RING - 1>();
    __syncwarp();
    unsigned char* slot = ring[(i + 2) % S_RING];
    swar_enter<NP, SYM>(slot, w, c - NP * lane, lane, a, H[S]);
    __syncwarp();
    if (i + 2 + S_RING < r_end) swar_issue<NP>(sw.src > sw.src_last ? sw.src_last : sw.src, slot, lane, body, halo);
    cp_commit();
    sw.src += sw.w;
    unsigned o[NP / 2];
#pragma unroll
    for (int t = 0; t < NP / 2; t++) {
        if (SYM) {  // u mirror-symmetric: rows i-2 / i+2 and i-1 / i+1 share a tap
            o[t] = a.half2 + a.u[0] * (H[(S + 1) % 5][t] + H[(S + 5) % 5][t]) +
                   a.u[1] * (H[(S + 2) % 5][t] + H[(S + 4) % 5][t]) + a.u[2] * H[(S + 3) % 5][t];
        } else {
            unsigned acc = a.half2;
#pragma unroll
            for (int di = 0; di < 5; di++) acc += a.u[di] * H[(S + 1 + di) % 5][t];
            o[t] = acc;
        }
    }
    unsigned char* orow = sw.dst;
    sw.dst += sw.w;
    unsigned r[NP / 4];
#pragma unroll
    for (int g = 0; g < NP / 4; g++) {
        if (SH8)  // the output bytes are the high bytes of the 16-bit lanes
            r[g] = __byte_perm(o[2 * g], o[2 * g + 1], 0x7351);
        else
            r[g] = ((o[2 * g] >> a.shift) & 0x00ff00ffu) | (((o[2 * g + 1] >> a.shift) & 0x00ff00ffu) << 8);
    }
    swar_store_if<NP>(body, orow, r);
}

// lo / hi: the output rows computed (the whole image: 0 / h; the pipelined drop-in: a row block)
template <int NP, bool SH8, bool SYM>
__device__ __forceinline__ void swar_sweep(int h, int w, const unsigned char* __restrict__ img,
                                           unsigned char* __restrict__ out, const SwarArgs& a, int lo, int hi) {
    typedef SwarGeom<NP> G;
    __shared__ __align__(16) unsigned char ring_all[S_WARPS][S_RING][G::ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = (blockIdx.x * S_WARPS + warp) * 32 * NP;
    if (c0 >= w) return;
    const int c = c0 + NP * lane;
    const int i0 = lo + blockIdx.y * S_BAND, i1 = min(hi, i0 + S_BAND);
    if (i0 >= i1) return;
    const int r_end = i1 + 2;
    const bool body = c + NP - 1 < w;
    const bool halo = (lane == 0 && c0 > 0) || (lane == 31 && c0 + 32 * NP < w);
    unsigned char(*ring)[G::ROWE] = ring_all[warp];
    auto row = [&](int r) { return img + (long long)clampi(r, 0, h - 1) * w + c; };
#pragma unroll
    for (int d = 0; d < S_RING; d++) {
        if (i0 - 2 + d < r_end) swar_issue<NP>(row(i0 - 2 + d), ring[(i0 - 2 + d + S_RING) % S_RING], lane, body, halo);
        cp_commit();
    }
    unsigned H[5][NP / 2];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        cp_wait<S_RING - 1>();
        __syncwarp();
        unsigned char* slot = ring[(i0 - 2 + d + S_RING) % S_RING];
        swar_enter<NP, SYM>(slot, w, c0, lane, a, H[d]);
        __syncwarp();
        if (i0 - 2 + d + S_RING < r_end) swar_issue<NP>(row(i0 - 2 + d + S_RING), slot, lane, body, halo);
        cp_commit();
    }
    Sweep<unsigned char> sw;
    sw.w = w;
    sw.src_last = img + (long long)(h - 1) * w + c;
    sw.src = img + (long long)(i0 + 2 + S_RING) * w + c;
    sw.dst = out + (long long)i0 * w + c;
    for (int i = i0; i < i1; i += 5) {
        swar_step<NP, 4, SH8, SYM>(w, i, c, lane, r_end, body, halo, ring, H, sw, a);
        if (i + 1 < i1) swar_step<NP, 0, SH8, SYM>(w, i + 1, c, lane, r_end, body, halo, ring, H, sw, a);
        if (i + 2 < i1) swar_step<NP, 1, SH8, SYM>(w, i + 2, c, lane, r_end, body, halo, ring, H, sw, a);
        if (i + 3 < i1) swar_step<NP, 2, SH8, SYM>(w, i + 3, c, lane, r_end, body, halo, ring, H, sw, a);
        if (i + 4 < i1) swar_step<NP, 3, SH8, SYM>(w, i + 4, c, lane, r_end, body, halo, ring, H, sw, a);
    }
    cp_wait<0>();
}
// the whole image (its own kernel: the row-block form's two extra parameters cost the sweep ~2 %)
template <int NP, bool SH8, bool SYM = false>
__global__ void __launch_bounds__(32 * S_WARPS, 4) stencil_bytes_swar_kernel(int h, int w,
                                                                           const unsigned char* __restrict__ img,
                                                                           unsigned char* __restrict__ out,
                                                                           SwarArgs a) {
    swar_sweep<NP, SH8, SYM>(h, w, img, out, a, 0, h);
}
// output rows [lo, hi) (the pipelined drop-in's row blocks)
template <int NP, bool SH8, bool SYM = false>
__global__ void __launch_bounds__(32 * S_WARPS, 4) stencil_bytes_swar_rows_kernel(int h, int w,
                                                                                const unsigned char* __restrict__ img,
                                                                                unsigned char* __restrict__ out,
                                                                                SwarArgs a, int lo, int hi) {
    swar_sweep<NP, SH8, SYM>(h, w, img, out, a, lo, hi);
}

// ---------------------------------------------------------------- signed 2-D SWAR packed-byte sweep
// Taps with a non-negative centre and non-positive off-centre taps (sharpen, Laplacian and
// unsharp-mask shapes — the signed sharpen of the config), power-of-two scale.  With
// B = 255 * sum |k_off| every 16-bit SWAR lane accumulates
//   acc = scale/2 + B + kc x_c - sum |k| x
// starting from scale/2 + B: each off-centre product is SUBTRACTED (an IMAD by the two's-complement
// tap k = -|k|, exact mod 2^32), and because the partial sums of |k| x never exceed B no lane ever
// borrows from its neighbour; when 255 * (kc + sum |k_off|) + scale / 2 < 65536 the lane never
// carries either.  One IMAD per tap per two pixels, no complement, no int -> float conversion.
// Requantisation per lane: (max(acc, B) - B) >> shift, then min 255 (C truncation and the [0, 255]
// clamp: a negative numerator gives 0 either way).  Rows are pushed: the row entering the window
// adds its taps to the five output rows it feeds (5 x NP/2 accumulators), and the output row it
// completes is requantised and stored.  Integer arithmetic throughout: bit-identical to the other
// kernels.
// DIA: the 12 corner taps are zero (skipped at compile time).
// SYM: taps mirror-symmetric in both axes (k[i][j] = k[4-i][j] = k[i][4-j]: sharpen, Laplacian,
// Gaussian shapes): per pixel pair the entering row forms the horizontal pair sums S1, S2 once,
// rows 0 / 4 and 1 / 3 share one partial each, so a diamond costs 6 IMADs + 6 adds per pair
// instead of 13 IMADs (the IMAD pipe runs at half the issue rate).
struct Swar2dArgs {
    unsigned kc;         // centre tap (>= 0)
    unsigned kn[25];     // off-centre taps as 32-bit two's complement (-|k|; kn[12] unused)
    unsigned init2;      // scale / 2 + B in both 16-bit lanes (the accumulators' start)
    unsigned bias2;      // B in both lanes
    int shift;           // log2(scale) <= 8
};

__device__ __forceinline__ unsigned umax16x2(unsigned a, unsigned b) {
    unsigned r;
    asm("max.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ unsigned umin16x2(unsigned a, unsigned b) {
    unsigned r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}

template <bool DIA>
__device__ __forceinline__ constexpr bool tap_on(int di, int dj) {
    return !DIA || ((di > 2 ? di - 2 : 2 - di) + (dj > 2 ? dj - 2 : 2 - dj) <= 2);
}

// Row r (slot S = r mod 5 of the rotation) enters: A[(r - di + 2) mod 5] += taps of row di.
// Then output row r - 2 is complete: requantise, store (when it lies in [i0, i1)), reset.
// EDGE: the warp may own an image-edge strip (clamped columns); STEADY: row r + S_RING is still
// an input row of the band and output row r - 2 lies in it (the sweep's middle: no row checks).
template <int NP, int S, bool DIA, bool SH0, bool SYM, bool EDGE, bool STEADY>
__device__ __forceinline__ void swar2d_step(int w, int r, int i0, int i1, int c, int lane, int r_end, bool body,
                                            bool halo, unsigned char (*ring)[SwarGeom<NP>::ROWE],
                                            unsigned (&A)[5][NP / 2], Sweep<unsigned char>& sw,
                                            const Swar2dArgs& a) {
    cp_wait<S_RING - 1>();
    __syncwarp();
    unsigned char* slot = ring[(r + S_RING) % S_RING];
    unsigned Q[NP + 2];
    swar_pairs<NP, EDGE>(slot, w, c - NP * lane, lane, Q);
    __syncwarp();
    if (STEADY || r + S_RING < r_end)
        swar_issue<NP>(sw.src > sw.src_last ? sw.src_last : sw.src, slot, lane, body, halo);
    cp_commit();
    sw.src += sw.w;
    if constexpr (SYM) {
        constexpr int o0 = (S + 7) % 5, o1 = (S + 6) % 5, o2 = (S + 5) % 5, o3 = (S + 4) % 5, o4 = (S + 3) % 5;
#pragma unroll
        for (int t = 0; t < NP / 2; t++) {
            const int b = (t & 1) + 4 * (t >> 1);
            const unsigned X = Q[b + 2], S1 = Q[b + 1] + Q[b + 3], S2 = Q[b] + Q[b + 4];
            unsigned H0 = X * a.kn[2], H1 = S1 * a.kn[6] + X * a.kn[7];
            if (!DIA) H0 += S2 * a.kn[0] + S1 * a.kn[1], H1 += S2 * a.kn[5];
            A[o0][t] += H0;
            A[o4][t] += H0;
            A[o1][t] += H1;
            A[o3][t] += H1;
            A[o2][t] += S2 * a.kn[10] + S1 * a.kn[11] + X * a.kc;
        }
    } else {
#pragma unroll
        for (int di = 0; di < 5; di++) {
            const int o = (S - di + 2 + 5) % 5;  // accumulator slot of output row r - di + 2
#pragma unroll
            for (int t = 0; t < NP / 2; t++) {
                const int b = (t & 1) + 4 * (t >> 1);
                unsigned acc = A[o][t];
#pragma unroll
                for (int dj = 0; dj < 5; dj++) {
                    if (!tap_on<DIA>(di, dj)) continue;
                    acc += (di == 2 && dj == 2 ? a.kc : a.kn[di * 5 + dj]) * Q[b + dj];
                }
                A[o][t] = acc;
            }
        }
    }
    // output row r - 2 (slot (S + 3) % 5 = (r - 2) mod 5) is complete
    constexpr int D = (S + 3) % 5;
    // (requantised unconditionally, stored under a predicate: no branch around the block)
    const int orow = r - 2;
    {
        unsigned q[NP / 2];
#pragma unroll
        for (int t = 0; t < NP / 2; t++) {
            unsigned v = umax16x2(A[D][t], a.bias2) - a.bias2;  // the numerator, clamped at 0
            if (!SH0) v = (v >> a.shift) & ((0xffffu >> a.shift) * 0x00010001u);  // scale 1: no shift
            q[t] = umin16x2(v, 0x00ff00ffu);
        }
        unsigned rr[NP / 4];
#pragma unroll
        for (int g = 0; g < NP / 4; g++) rr[g] = __byte_perm(q[2 * g], q[2 * g + 1], 0x6240);
        swar_store_if<NP>((STEADY || (orow >= i0 && orow < i1)) && body, sw.dst + (long long)(orow - i0) * w, rr);
    }
#pragma unroll
    for (int t = 0; t < NP / 2; t++) A[D][t] = a.init2;
}

// Rows r0, r0 + 5, ... while r < r_stop (and r < r_end), five steps per iteration; returns the
// first row not run.  STEADY callers pass r_stop so that every row of their iterations is
// in the band's middle.
template <int NP, bool DIA, bool SH0, bool SYM, bool EDGE, bool STEADY>
__device__ __forceinline__ int swar2d_rows(int r, int r_stop, int w, int i0, int i1, int c, int lane, int r_begin,
                                           int r_end, bool body, bool halo,
                                           unsigned char (*ring)[SwarGeom<NP>::ROWE], unsigned (&A)[5][NP / 2],
                                           Sweep<unsigned char>& sw, const Swar2dArgs& a) {
    for (; r < r_stop && r < r_end; r += 5) {
        if (STEADY) {
            swar2d_step<NP, 0, DIA, SH0, SYM, EDGE, true>(w, r + 0, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
            swar2d_step<NP, 1, DIA, SH0, SYM, EDGE, true>(w, r + 1, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
            swar2d_step<NP, 2, DIA, SH0, SYM, EDGE, true>(w, r + 2, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
            swar2d_step<NP, 3, DIA, SH0, SYM, EDGE, true>(w, r + 3, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
            swar2d_step<NP, 4, DIA, SH0, SYM, EDGE, true>(w, r + 4, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
            continue;
        }
#define SWAR2D_STEP(k)                                                                                         \
    if (r + k >= r_begin && r + k < r_end)                                                                     \
        swar2d_step<NP, k, DIA, SH0, SYM, EDGE, false>(w, r + k, i0, i1, c, lane, r_end, body, halo, ring, A, sw, a);
        SWAR2D_STEP(0) SWAR2D_STEP(1) SWAR2D_STEP(2) SWAR2D_STEP(3) SWAR2D_STEP(4)
#undef SWAR2D_STEP
    }
    return r;
}

template <int NP, bool DIA, bool SH0, bool SYM>
__device__ __forceinline__ void swar2d_sweep(int h, int w, const unsigned char* __restrict__ img,
                                             unsigned char* __restrict__ out, const Swar2dArgs& a, int lo, int hi) {
    typedef SwarGeom<NP> G;
    __shared__ __align__(16) unsigned char ring_all[S_WARPS][S_RING][G::ROWE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = (blockIdx.x * S_WARPS + warp) * 32 * NP;
    if (c0 >= w) return;
    const int c = c0 + NP * lane;
    const int i0 = lo + blockIdx.y * S_BAND, i1 = min(hi, i0 + S_BAND);
    if (i0 >= i1) return;
    const int r_begin = i0 - 2, r_end = i1 + 2;  // input rows of the band (clamped at the image edges)
    const bool body = c + NP - 1 < w;
    const bool halo = (lane == 0 && c0 > 0) || (lane == 31 && c0 + 32 * NP < w);
    unsigned char(*ring)[G::ROWE] = ring_all[warp];
    auto row = [&](int r) { return img + (long long)clampi(r, 0, h - 1) * w + c; };
#pragma unroll
    for (int d = 0; d < S_RING; d++) {
        if (r_begin + d < r_end) swar_issue<NP>(row(r_begin + d), ring[(r_begin + d + S_RING) % S_RING], lane, body, halo);
        cp_commit();
    }
    unsigned A[5][NP / 2];
#pragma unroll
    for (int q = 0; q < 5; q++)
#pragma unroll
        for (int t = 0; t < NP / 2; t++) A[q][t] = a.init2;
    Sweep<unsigned char> sw;
    sw.w = w;
    sw.src_last = img + (long long)(h - 1) * w + c;
    sw.src = img + (long long)(r_begin + S_RING) * w + c;
    sw.dst = out + (long long)i0 * w + c;
    // the rotation slot of row r is r mod 5; start at a multiple of 5 at or below r_begin so the
    // slots stay compile-time constants (rows before r_begin are skipped).  (A peeled middle
    // without row checks, and a separate copy for warps away from the image edges, measured
    // 0.193 / 0.229 ms against 0.156: three copies of the five-step body thrash the instruction
    // cache.)
    const int rb5 = r_begin - ((r_begin % 5) + 5) % 5;
    swar2d_rows<NP, DIA, SH0, SYM, true, false>(rb5, r_end, w, i0, i1, c, lane, r_begin, r_end, body, halo, ring, A,
                                                sw, a);
    cp_wait<0>();
}
template <int NP, bool DIA, bool SH0 = false, bool SYM = false>
__global__ void __launch_bounds__(32 * S_WARPS, 4) stencil_bytes_swar2d_kernel(int h, int w,
                                                                             const unsigned char* __restrict__ img,
                                                                             unsigned char* __restrict__ out,
                                                                             Swar2dArgs a) {
    swar2d_sweep<NP, DIA, SH0, SYM>(h, w, img, out, a, 0, h);
}
template <int NP, bool DIA, bool SH0 = false, bool SYM = false>
__global__ void __launch_bounds__(32 * S_WARPS, 4) stencil_bytes_swar2d_rows_kernel(int h, int w,
                                                                                  const unsigned char* __restrict__ img,
                                                                                  unsigned char* __restrict__ out,
                                                                                  Swar2dArgs a, int lo, int hi) {
    swar2d_sweep<NP, DIA, SH0, SYM>(h, w, img, out, a, lo, hi);
}

// Swar2dArgs for taps with kc >= 0, every off-centre tap <= 0, a power-of-two scale <= 256 and
// every biased sum below 2^16; false otherwise.
bool swar2d_args(const int* k, int scale, Swar2dArgs& a) {
#ifdef PENCIL_VARIANT_NO_SWAR
    return false;
#endif
    if (scale < 1 || scale > 256 || (scale & (scale - 1))) return false;
    if (k[12] < 0) return false;
    long long off = 0;
    for (int t = 0; t < 25; t++) {
        if (t == 12) continue;
        if (k[t] > 0) return false;
        off += -(long long)k[t];
    }
    const long long B = 255 * off;
    if (255ll * ((long long)k[12] + off) + (scale >> 1) >= 65536) return false;
    a.kc = (unsigned)k[12];
    for (int t = 0; t < 25; t++) a.kn[t] = t == 12 ? 0u : (unsigned)k[t];  // k <= 0: -|k| mod 2^32
    a.init2 = (unsigned)((scale >> 1) + B) * 0x00010001u;
    a.bias2 = (unsigned)B * 0x00010001u;
    a.shift = 0;
    while ((1 << a.shift) != scale) a.shift++;
    return true;
}

// taps mirror-symmetric in both axes
bool mirror_symmetric(const int* k) {
    for (int i = 0; i < 5; i++)
        for (int j = 0; j < 5; j++)
            if (k[i * 5 + j] != k[(4 - i) * 5 + j] || k[i * 5 + j] != k[i * 5 + 4 - j]) return false;
    return true;
}

// SwarArgs from the separable factorisation, or false (signs, sums >= 2^16, clamp needed).
// (A/B builds: tools/variant_build.sh compiles -DPENCIL_VARIANT_NO_SWAR into variants/.)
bool swar_args(const StencilArgs& s, int scale, SwarArgs& a) {
#ifdef PENCIL_VARIANT_NO_SWAR
    return false;
#endif
    if (s.shift < 0 || s.shift > 8) return false;
    long long u[5], v[5], su = 0, sv = 0;
    bool uneg = true, vneg = true;
    for (int t = 0; t < 5; t++) {
        u[t] = (long long)s.ku[t];
        v[t] = (long long)s.kv[t];
        uneg &= u[t] <= 0;
        vneg &= v[t] <= 0;
    }
    if (uneg && vneg)
        for (int t = 0; t < 5; t++) u[t] = -u[t], v[t] = -v[t];
    for (int t = 0; t < 5; t++) {
        if (u[t] < 0 || v[t] < 0) return false;
        su += u[t];
        sv += v[t];
    }
    const long long mx = 255ll * su * sv + (scale >> 1);
    if (mx > 65535 || (mx >> s.shift) > 255) return false;
    for (int t = 0; t < 5; t++) {
        a.u[t] = (unsigned)u[t];
        a.v[t] = (unsigned)v[t];
    }
    a.half2 = (unsigned)(scale >> 1) * 0x00010001u;
    a.shift = s.shift;
    return true;
}

// (A/B builds: -DPENCIL_VARIANT_NO_SEP disables the separable kernels)
bool sep_enabled() {
#ifdef PENCIL_VARIANT_NO_SEP
    return false;
#else
    return true;
#endif
}

// Taps supported on the radius-2 diamond (|di-2| + |dj-2| <= 2: the 12 corner taps zero — the
// isotropic sharpen / Laplacian shapes): the DIA kernels skip the zero taps at compile time
// (13 FFMA2 per pixel pair instead of 25; exact integer sums, so bit-identical).
// (A/B builds: -DPENCIL_VARIANT_NO_DIA disables them.)
bool diamond(const int* k) {
#ifdef PENCIL_VARIANT_NO_DIA
    return false;
#endif
    for (int di = 0; di < 5; di++)
        for (int dj = 0; dj < 5; dj++)
            if (abs(di - 2) + abs(dj - 2) > 2 && k[di * 5 + dj]) return false;
    return true;
}

unsigned* repair_flag_for(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, unsigned*> flags;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    unsigned*& f = flags[{dev, st}];
    if (!f) {
        if (cudaMalloc(&f, 4 * sizeof(unsigned)) != cudaSuccess) {  // [0] u8, [2..3] f32 PF
            f = nullptr;
            return nullptr;
        }
        cudaMemset(f, 0, 4 * sizeof(unsigned));  // synchronous: before any launch can read it
    }
    return f;
}

// conv5x5_f32 taps whose products are exact: fusing `acc + k*x` into one FMA is then the same
// single rounding as the emitted C's rounded product + rounded sum.  A tap qualifies when it is
// 0 or +-2^e with -126 <= e <= 0 (no overflow; k*x exact unless it lands below 2^-126, which the
// kernel's guard catches: pixels with 0 < |x| < 2^(-126 - emin) divert the launch to the exact
// pass).  Returns the PF pattern (2: all 25 taps, 1: the 16 off the centre row/column, 0: none)
// and the guard's limit.  (A/B builds: -DPENCIL_VARIANT_NO_PF disables it.)
bool pow2_tap(float k, int& e) {
    unsigned u;
    memcpy(&u, &k, 4);
    u &= 0x7fffffffu;
    if (u == 0) return true;
    if ((u & 0x7fffffu) != 0) return false;
    const int ex = (int)(u >> 23) - 127;
    if (ex < -126 || ex > 0) return false;
    e = ex < e ? ex : e;
    return true;
}
int pow2_fusable(const float* k25, unsigned& lim) {
#ifdef PENCIL_VARIANT_NO_PF
    return 0;
#endif
    for (int pf = 2; pf >= 1; pf--) {
        int emin = 0;
        bool ok = true;
        for (int di = 0; di < 5 && ok; di++)
            for (int dj = 0; dj < 5 && ok; dj++)
                if (pf_tap(pf, di, dj)) ok = pow2_tap(k25[di * 5 + dj], emin);
        if (ok) {
            lim = ((unsigned)(1 - emin) << 23) - 1u;  // bits of 2^(-126 - emin), minus 1
            return pf;
        }
    }
    return 0;
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
    StencilArgsF32 a = {};
    for (int t = 0; t < 25; t++) a.kf[t] = k25[t];
    a.negz = pack2(-0.0f);
    a.one = pack2(1.0f);
    a.negmag = pack2(-8388608.0f);
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h - 4 + ring_band<false>() - 1) / ring_band<false>());
    const int pf = pow2_fusable(k25, a.pf_lim);
    unsigned* flag = pf ? repair_flag_for(st) : nullptr;
    if (pf && flag) {
        a.repair_flag = flag + 2;
        if (pf == 2)
            stencil_ring_kernel<false, false, false, false, 2><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else
            stencil_ring_kernel<false, false, false, false, 1><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        f32_repair_kernel<<<PENCIL_NUM_SMS * 4, 256, 0, st>>>(h, w, img, out, a);
    } else {
        stencil_ring_kernel<false, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    }
    return (int)cudaGetLastError();
}

namespace {
// conv5x5_u8 launch arguments: taps, requantisation constants, the stream's repair flag
bool u8_args(cudaStream_t st, int scale, const int* k25, StencilArgs& a) {
    bool small = true;
    for (int t = 0; t < 25; t++) {
        a.kf[t] = (float)k25[t];
        a.ki[t] = k25[t];
        small &= (k25[t] >= -657 && k25[t] <= 657);  // |acc| <= 25 * 255 * 657 < 2^22
    }
    a.exact_only = small ? 0 : 1;
    a.negz = pack2(-0.0f);
    a.one = pack2(1.0f);
    a.negmag = pack2(-8388608.0f);
    a.scale = scale;
    a.shift = -1;
    if (scale > 0 && (scale & (scale - 1)) == 0) {
        a.shift = 0;
        while ((1 << a.shift) != scale) a.shift++;
        a.inv_scale = pack2(ldexpf(1.0f, -a.shift));
        a.half_scaled = pack2((float)(scale >> 1) * ldexpf(1.0f, -a.shift));
        a.magic2 = pack2(12582912.0f);
    } else if (scale >= 2) {
        a.magic = ~0ull / (unsigned long long)scale + 1;
    }
    // repair flag per (device, stream): zero between launches (the repair pass re-arms it), and
    // launches on different streams never see each other's flag
    a.repair_flag = repair_flag_for(st);
    return a.repair_flag != nullptr;
}
}  // namespace

int launch_conv5x5_u8(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25, int* out) {
    if (h <= 0 || w <= 0) return 0;
    if (!ring_ok(h, w, img, out)) return launch_conv5x5_u8_reg(st, h, w, scale, img, k25, out);
    StencilArgs a = {};
    if (!u8_args(st, scale, k25, a)) return (int)cudaErrorMemoryAllocation;
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h + ring_band<true>() - 1) / ring_band<true>());
    if (!a.exact_only) {
        const bool sep = sep_enabled() && separable(k25, a), dia = !sep && diamond(k25);
        if (sep && a.shift >= 0) stencil_ring_kernel<true, true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else if (sep) stencil_ring_kernel<true, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else if (dia && a.shift >= 0) stencil_ring_kernel<true, true, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else if (dia) stencil_ring_kernel<true, false, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else if (a.shift >= 0) stencil_ring_kernel<true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
        else stencil_ring_kernel<true, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    }
    const long long n = (long long)h * w, blocks = (n + 255) / 256;
    u8_repair_kernel<<<(int)(blocks < PENCIL_NUM_SMS * 8 ? blocks : PENCIL_NUM_SMS * 8), 256, 0, st>>>(h, w, img, out, a);
    u8_rearm_kernel<<<1, 1, 0, st>>>(a.repair_flag);
    return (int)cudaGetLastError();
}

// Band-sharded launches (the fused halo exchange): `top` / `bot` hold the row pointers of rows
// -2, -1 and h, h + 1 of the band (see BandSrc).  Need w % 4 == 0 and 16-byte aligned rows.
static bool band_ok(int h, int w, const void* img, const void* out, const void* const* top, const void* const* bot) {
    bool ok = ring_ok(h, w, img, out);
    for (int t = 0; t < 2; t++) ok = ok && top[t] && bot[t] && (uintptr_t)top[t] % 16 == 0 && (uintptr_t)bot[t] % 16 == 0;
    return ok;
}

int launch_conv5x5_u8_band(cudaStream_t st, int h, int w, int scale, const int* img, const int* const* top,
                           const int* const* bot, const int* k25, int* out) {
    if (h <= 0 || w <= 0) return 0;
    if (!band_ok(h, w, img, out, (const void* const*)top, (const void* const*)bot)) return (int)cudaErrorInvalidValue;
    StencilArgs a = {};
    if (!u8_args(st, scale, k25, a)) return (int)cudaErrorMemoryAllocation;
    const BandSrc<int> bs = {{top[0], top[1]}, {bot[0], bot[1]}, 0, h};
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h + ring_band<true>() - 1) / ring_band<true>());
    if (!a.exact_only) {
        const bool sep = sep_enabled() && separable(k25, a), dia = !sep && diamond(k25);
        if (sep && a.shift >= 0) stencil_band_kernel<true, true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else if (sep) stencil_band_kernel<true, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else if (dia && a.shift >= 0) stencil_band_kernel<true, true, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else if (dia) stencil_band_kernel<true, false, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else if (a.shift >= 0) stencil_band_kernel<true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else stencil_band_kernel<true, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
    }
    const long long n = (long long)h * w, blocks = (n + 255) / 256;
    u8_band_repair_kernel<<<(int)(blocks < PENCIL_NUM_SMS * 8 ? blocks : PENCIL_NUM_SMS * 8), 256, 0, st>>>(h, w, img, out, a, bs);
    u8_rearm_kernel<<<1, 1, 0, st>>>(a.repair_flag);
    return (int)cudaGetLastError();
}

int launch_conv5x5_f32_band(cudaStream_t st, int h, int w, int out_lo, int out_hi, const float* img,
                            const float* const* top, const float* const* bot, const float* k25, float* out) {
    if (h <= 0 || w < 5 || out_lo >= out_hi) return 0;
    if (out_lo < 0 || out_hi > h) return (int)cudaErrorInvalidValue;
    if (!band_ok(h, w, img, out, (const void* const*)top, (const void* const*)bot)) return (int)cudaErrorInvalidValue;
    StencilArgsF32 a = {};
    for (int t = 0; t < 25; t++) a.kf[t] = k25[t];
    a.negz = pack2(-0.0f);
    a.one = pack2(1.0f);
    a.negmag = pack2(-8388608.0f);
    const BandSrc<float> bs = {{top[0], top[1]}, {bot[0], bot[1]}, out_lo, out_hi};
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (out_hi - out_lo + ring_band<false>() - 1) / ring_band<false>());
    // power-of-two taps fused as in launch_conv5x5_f32, with the band's own guarded repair pass
    const int pf = pow2_fusable(k25, a.pf_lim);
    unsigned* flag = pf ? repair_flag_for(st) : nullptr;
    if (pf && flag) {
        a.repair_flag = flag + 2;
        if (pf == 2)
            stencil_band_kernel<false, false, false, false, 2><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        else
            stencil_band_kernel<false, false, false, false, 1><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
        f32_band_repair_kernel<<<PENCIL_NUM_SMS * 4, 256, 0, st>>>(h, w, img, out, a, bs);
    } else {
        stencil_band_kernel<false, false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, bs);
    }
    return (int)cudaGetLastError();
}

int launch_conv5x5_u8_bytes_dp4a(cudaStream_t st, int h, int w, int scale, const unsigned char* img,
                                 const int* k25, unsigned char* out);

// the whole-image kernel, or its row-block twin
template <typename Arg>
static void swar_go(void (*kw)(int, int, const unsigned char*, unsigned char*, Arg),
                    void (*kr)(int, int, const unsigned char*, unsigned char*, Arg, int, int), dim3 g,
                    cudaStream_t st, bool rows, int h, int w, const unsigned char* img, unsigned char* out,
                    const Arg& a, int lo, int hi) {
    if (rows) kr<<<g, 32 * S_WARPS, 0, st>>>(h, w, img, out, a, lo, hi);
    else kw<<<g, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
}
// Output rows [lo, hi) of the h-row image (rows_only: only when a SWAR kernel applies — the row-block
// form of the pipelined drop-in; returns cudaErrorNotSupported otherwise, launching nothing).
// probe: report whether the row-block form applies (16-byte aligned buffers assumed), launch nothing.
static int conv_u8_bytes_rows(cudaStream_t st, int h, int w, int scale, const unsigned char* img, const int* k25,
                              unsigned char* out, int lo, int hi, bool rows_only, bool probe = false);
int launch_conv5x5_u8_bytes(cudaStream_t st, int h, int w, int scale, const unsigned char* img, const int* k25,
                            unsigned char* out) {
    return conv_u8_bytes_rows(st, h, w, scale, img, k25, out, 0, h, false);
}
int launch_conv5x5_u8_bytes_rows(cudaStream_t st, int h, int w, int scale, const unsigned char* img, const int* k25,
                                 unsigned char* out, int lo, int hi) {
    if (lo < 0 || hi > h || lo > hi) return (int)cudaErrorInvalidValue;
    return conv_u8_bytes_rows(st, h, w, scale, img, k25, out, lo, hi, true);
}
bool conv5x5_u8_bytes_rows_ok(int h, int w, int scale, const int* k25) {
    return h > 0 && conv_u8_bytes_rows(nullptr, h, w, scale, nullptr, k25, nullptr, 0, h, true, true) == 0;
}
static int conv_u8_bytes_rows(cudaStream_t st, int h, int w, int scale, const unsigned char* img, const int* k25,
                              unsigned char* out, int lo, int hi, bool rows_only, bool probe) {
    if (h <= 0 || w <= 0 || hi <= lo) return probe ? (int)cudaErrorNotSupported : 0;
    bool small = true;
    for (int t = 0; t < 25; t++) small &= (k25[t] >= -657 && k25[t] <= 657);
    if (!small || w % 4 != 0 || (uintptr_t)img % 4 != 0 || (uintptr_t)out % 4 != 0)
        return rows_only ? (int)cudaErrorNotSupported : launch_conv5x5_u8_bytes_dp4a(st, h, w, scale, img, k25, out);
    StencilArgs a = {};
    for (int t = 0; t < 25; t++) {
        a.kf[t] = (float)k25[t];
        a.ki[t] = k25[t];
    }
    a.negz = pack2(-0.0f);
    a.one = pack2(1.0f);
    a.negmag = pack2(-8388608.0f);
    a.scale = scale;
    a.shift = -1;
    if (scale > 0 && (scale & (scale - 1)) == 0) {
        a.shift = 0;
        while ((1 << a.shift) != scale) a.shift++;
        a.inv_scale = pack2(ldexpf(1.0f, -a.shift));
        a.half_scaled = pack2((float)(scale >> 1) * ldexpf(1.0f, -a.shift));
        a.magic2 = pack2(12582912.0f);
    } else if (scale >= 2) {
        a.magic = ~0ull / (unsigned long long)scale + 1;
    }
    dim3 grid(((w + 127) / 128 + S_WARPS - 1) / S_WARPS, (h + S_BAND - 1) / S_BAND);
    const bool sep = sep_enabled() && separable(k25, a), dia = !sep && diamond(k25);
    SwarArgs sa;
    Swar2dArgs s2;
    if (sep && w % 8 == 0 && (uintptr_t)img % 8 == 0 && (uintptr_t)out % 8 == 0 && swar_args(a, scale, sa)) {
#ifdef PENCIL_VARIANT_SWAR_NP8
        const int np_max = 8;
#else
        const int np_max = 16;
#endif
        const bool n16 = np_max == 16 && w % 16 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0;
        const int np = n16 ? 16 : 8;
        dim3 g(((w + 32 * np - 1) / (32 * np) + S_WARPS - 1) / S_WARPS, (hi - lo + S_BAND - 1) / S_BAND);
        const bool sym = sa.u[0] == sa.u[4] && sa.u[1] == sa.u[3] && sa.v[0] == sa.v[4] && sa.v[1] == sa.v[3];
        if (probe) return 0;
        if (n16 && sym && sa.shift == 8)
            swar_go<SwarArgs>(stencil_bytes_swar_kernel<16, true, true>, stencil_bytes_swar_rows_kernel<16, true, true>, g, st, rows_only, h, w, img, out, sa, lo, hi);
        else if (n16 && sym) swar_go<SwarArgs>(stencil_bytes_swar_kernel<16, false, true>, stencil_bytes_swar_rows_kernel<16, false, true>, g, st, rows_only, h, w, img, out, sa, lo, hi);
        else if (n16 && sa.shift == 8) swar_go<SwarArgs>(stencil_bytes_swar_kernel<16, true>, stencil_bytes_swar_rows_kernel<16, true>, g, st, rows_only, h, w, img, out, sa, lo, hi);
        else if (n16) swar_go<SwarArgs>(stencil_bytes_swar_kernel<16, false>, stencil_bytes_swar_rows_kernel<16, false>, g, st, rows_only, h, w, img, out, sa, lo, hi);
        else if (sa.shift == 8) swar_go<SwarArgs>(stencil_bytes_swar_kernel<8, true>, stencil_bytes_swar_rows_kernel<8, true>, g, st, rows_only, h, w, img, out, sa, lo, hi);
        else swar_go<SwarArgs>(stencil_bytes_swar_kernel<8, false>, stencil_bytes_swar_rows_kernel<8, false>, g, st, rows_only, h, w, img, out, sa, lo, hi);
    } else if (!sep && w % 8 == 0 && (uintptr_t)img % 8 == 0 && (uintptr_t)out % 8 == 0 &&
               swar2d_args(k25, scale, s2)) {
        const bool n16 = w % 16 == 0 && (uintptr_t)img % 16 == 0 && (uintptr_t)out % 16 == 0;
        const int np = n16 ? 16 : 8;
        dim3 g(((w + 32 * np - 1) / (32 * np) + S_WARPS - 1) / S_WARPS, (hi - lo + S_BAND - 1) / S_BAND);
        if (probe) return 0;
        const bool sym = mirror_symmetric(k25);
        if (n16 && sym && dia && s2.shift == 0)
            swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, true, true, true>, stencil_bytes_swar2d_rows_kernel<16, true, true, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (n16 && sym && dia)
            swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, true, false, true>, stencil_bytes_swar2d_rows_kernel<16, true, false, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (n16 && sym)
            swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, false, false, true>, stencil_bytes_swar2d_rows_kernel<16, false, false, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (n16 && dia && s2.shift == 0)
            swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, true, true>, stencil_bytes_swar2d_rows_kernel<16, true, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (n16 && dia) swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, true>, stencil_bytes_swar2d_rows_kernel<16, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (n16) swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<16, false>, stencil_bytes_swar2d_rows_kernel<16, false>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else if (dia) swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<8, true>, stencil_bytes_swar2d_rows_kernel<8, true>, g, st, rows_only, h, w, img, out, s2, lo, hi);
        else swar_go<Swar2dArgs>(stencil_bytes_swar2d_kernel<8, false>, stencil_bytes_swar2d_rows_kernel<8, false>, g, st, rows_only, h, w, img, out, s2, lo, hi);
    } else if (rows_only) {
        return (int)cudaErrorNotSupported;
    } else if (sep && a.shift >= 0) stencil_bytes_kernel<true, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    else if (sep) stencil_bytes_kernel<false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    else if (dia && a.shift >= 0) stencil_bytes_kernel<true, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    else if (dia) stencil_bytes_kernel<false, false, true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    else if (a.shift >= 0) stencil_bytes_kernel<true><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    else stencil_bytes_kernel<false><<<grid, 32 * S_WARPS, 0, st>>>(h, w, img, out, a);
    return (int)cudaGetLastError();
}
