// conv5x5_u8 on packed 8-bit storage (1 byte per pixel in and out): same semantics as
// conv5x5_u8 (clamp-to-edge, (acc + scale/2)/scale truncating, saturate).  A lane owns 16
// pixels (one uint4); window rows are 6 words (own 4 + the neighbours' edge words by shuffle);
// each pixel is 10 dp4a.u32.s32 against pre-shifted tap words (no byte extraction).  Taps
// outside int8 take the per-pixel int32 path.  IDP4A-bound (~0.5 ms at 16384^2).
#include "common.cuh"
#include "kernels.h"

namespace {

#define CONV_BAND 64
#define CONV_WARPS 4

struct TapsI { int k[25]; };
struct TapsDp4a { unsigned w[5][4][2]; };
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

}  // namespace

// the packed-u8 ring kernel (k_stencil.cu) is the default; this is its fallback for taps
// with |k| > 657 and layouts it does not take
int launch_conv5x5_u8_bytes_dp4a(cudaStream_t st, int h, int w, int scale, const unsigned char* img,
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
