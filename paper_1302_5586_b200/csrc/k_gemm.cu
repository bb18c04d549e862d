// gemm.pencil.c on the 5th-generation tensor cores: C = alpha * A B + beta * C in fp32 via
// 3xTF32 (tcgen05.mma kind::tf32, accumulators in TMEM, operands staged by TMA).
//
// Schedule (mapper): i, j ASSUMED_PARALLEL -> 2-D grid of 256 x 256 output tiles, one per CTA
// pair; p PARALLEL_WITH_REDUCTION(+) -> the K loop is split across tensor-core MMAs (reassociates).
//
// Precision: x = hi + lo with hi = x truncated to tf32 (the tensor core reads only the sign,
// exponent and top 10 mantissa bits of a 32-bit operand, so the raw fp32 tile IS the hi operand)
// and lo = rna_tf32(x - hi) (x - hi is exact: at most the 13 dropped bits).  The kernel
// accumulates lo*hi + hi*lo + hi*hi in fp32 (TMEM); the dropped lo*lo term (< 2^-20 |ab|) and the
// tf32 rounding of lo (< 2^-22 |x|) stay well inside the 1e-5 normwise tolerance of the tests.
//
// No prologue, no workspace: A (M x K row-major) is read in place as a K-major operand, B (K x N
// row-major) in place as an MN-major operand (tcgen05 takes tf32 in either major), both by TMA
// straight from the caller's arrays; ragged M / N / K edges are zero-filled by the TMA unit.  Only
// the lo halves are derived, on chip: per stage a converter warpgroup reads the 16 KB hi tile out
// of shared memory and writes its lo twin next to it (elementwise, so the swizzled layout carries
// over).  Operands whose row pitch is not a multiple of 16 bytes are first copied to a padded
// pitch (`pack_rows_kernel`; the only case that needs a workspace).
//
// Kernel anatomy (persistent: one CTA pair per two SMs, tiles handed out statically in a grouped
// raster; 10 warps per CTA):
//   warp 0    TMA producer (both CTAs): per K block of 16, A box 128x16 (K-major, SW64) and four
//             B boxes 32x16 (MN-major, SW128 with 32 B atoms) into a 6-stage ring of 32 KB (hi 16 KB + lo 16 KB),
//             completion on the CTA's own `full` mbarrier
//   warps 2-5 converters (both CTAs): wait `full`, lo = rna(x - trunc(x)) over the stage's hi
//             bytes, fence.proxy.async, one arrive per warp on the leader's `conv` barrier
//   warp 1    (leader CTA) TMEM allocator + MMA issuer (one elected lane): per K block 2 k-steps x
//             3 products tcgen05.mma.cta_group::2.kind::tf32 256x256x8 into one of two TMEM
//             accumulators (2 x 256 columns), tcgen05.commit multicast -> both CTAs' `empty`;
//             after the tile's last block, commit -> `tmem_full`
//   warps 6-9 epilogue (both CTAs): tcgen05.ld 32x32b.x32 (TMEM lane quarter = warp % 4) ->
//             alpha, beta -> 128-bit stores, then one arrive per warp on the leader's
//             `tmem_empty` — so tile t's epilogue overlaps tile t+1's main loop.
//
// Measured (16384^3 / 8192^3, tools/gemm_ab.sh): round 1's split prologue + 2-CTA kernel 37.4 ms
// (1.39 ms of it the split kernels); this kernel 34.6-36.5 ms (box to box) / 3.77 ms = 291 TFLOP/s,
// tensor pipe 97.8 % of active cycles at the power-capped 1.50 GHz.  Its first build ran 54 ms —
// unchanged with one MMA per k-step instead of three (so not tensor-bound), 39 ms with the converter
// loop removed: the converter used generic LD/ST on shared addresses and `.release.cluster` remote
// arrives (MEMBAR.ALL.GPU + ERRBAR per arrive); explicit ld/st.shared.v4 and default-semantics
// arrives fixed it.  (Those were timing-only builds with wrong results, not kept.)  A nanosleep
// back-off in the epilogue's wait for its accumulator (to spend fewer issue slots under the power
// cap) measured the same: 36.3-36.9 ms either way on one box.  The converters' power matters:
// without the cvt.rna.tf32 (lo left for the tensor core to truncate, -DGEMM_LO_TRUNC) the kernel
// ran 2.7 % faster (34.2 -> 33.3 ms, 16384^3, same box) at twice the error bound; lo_tf32 now gets
// the same round-to-nearest from one integer add (the tensor core's truncation does the rest):
// bit-identical C (tools/gemm_bits.py, 1536x1280x2064 and 4096^3) and 1.7 % faster than the CVT
// (35.0 / 35.6 vs 35.6 / 36.3 ms at 16384^3 on one box, 3.72 vs 3.75 ms at 8192^3).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace {

constexpr int BK = 16;                   // fp32 per K block: 64-byte A rows (swizzle-64B)
constexpr int TILE_M = 256, TILE_N = 256;  // per CTA pair
constexpr int CTA_M = 128, CTA_N = 128;    // A rows / B columns staged by each CTA of the pair
constexpr int A_BYTES = CTA_M * BK * 4;    // 8 KB
constexpr int B_CHUNK = 32;                // B columns per 128-byte swizzle row
constexpr int B_CHUNK_BYTES = B_CHUNK * BK * 4;  // 2 KB (16 K rows x 128 B)
constexpr int B_BYTES = CTA_N * BK * 4;    // 8 KB = 4 chunks
constexpr int HI_BYTES = A_BYTES + B_BYTES;
constexpr int STAGE_BYTES = 2 * HI_BYTES;  // hi | lo
constexpr int STAGES = 6;
constexpr int GEMM_THREADS = 320;
constexpr int CONV_WARP0 = 2, EPI_WARP0 = 6;
constexpr int TMEM_COLS = 512;  // two 256-column fp32 accumulators
constexpr int NUM_BARS = 3 * STAGES + 4;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + NUM_BARS * 8 + 16;
#ifndef GEMM_GROUP_M_DEF
#define GEMM_GROUP_M_DEF 8  // raster group in 256-row tiles (round 1 sweep 2/4/8/16: 8 best; round 2 re-check
                            // on the fused kernel: 4 / 8 / 16 -> 33.7-34.4 / 33.2-33.4 / 33.4-33.5 ms at 16384^3)
#endif
constexpr int GROUP_M = GEMM_GROUP_M_DEF;

// idesc: D fp32 (bit 4), A tf32 [7,10), B tf32 [10,13), A K-major (bit 15 = 0), B MN-major
// (bit 16 = 1), N >> 3 at [17,23), M >> 4 at [24,29)
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(TILE_N >> 3) << 17) |
                           ((uint32_t)(TILE_M >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// arrive on the same barrier in the leader CTA (cluster rank 0) — local for the leader itself.
// Default (.release.cta) semantics, as the arrive that hands a stage to the MMA: a .cluster
// release compiles to MEMBAR.ALL.GPU + ERRBAR per arrive and made the converters the bottleneck.
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* b) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(smem_u32(b)));
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// A: K-major, 64-byte swizzle: 8-row atoms of 8 x 64 B stacked every 512 B (SBO)
__device__ __forceinline__ uint64_t desc_a(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;     // SBO: next 8-row atom
    d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
    d |= (uint64_t)4 << 61;              // SWIZZLE_64B
    return d;
}
// B: MN-major.  tf32 MN-major operands take only the 128-byte swizzle with 32-byte atoms
// (SWIZZLE_128B_BASE32B: 128 B rows of 32 columns, one per k, the four 32 B granules of a row
// permuted by (row mod 4) — TMA's SWIZZLE_128B_ATOM_32B): 4-k atoms every 512 B (SBO), 32-column
// chunks every 2 KB (LBO)
__device__ __forceinline__ uint64_t desc_b(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)(B_CHUNK_BYTES >> 4) << 16;  // LBO: next 32-column chunk
    d |= (uint64_t)(512 >> 4) << 32;            // SBO: next 4 k
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;                     // SWIZZLE_128B_BASE32B
    return d;
}
__device__ __forceinline__ void mma_tf32_2sm(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void commit_2sm(uint64_t* bar) {  // arrive on bar in both CTAs
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// lo = rna_tf32(x - hi), as the tensor core will read it: it keeps the sign, exponent and top 10
// mantissa bits of a 32-bit operand (truncation), so adding half a tf32 ulp to the magnitude bits
// (+0x1000; a carry into the exponent is the correct round-up) makes its truncation round to
// nearest, ties away — the value cvt.rna.tf32.f32 gives, for one integer add instead of the CVT.
__device__ __forceinline__ uint32_t lo_tf32(uint32_t x) {
    const float r = __uint_as_float(x) - __uint_as_float(x & 0xffffe000u);  // exact
#if defined(GEMM_LO_TRUNC)  // A/B build: lo left for the tensor core to truncate
    return __float_as_uint(r);
#elif defined(GEMM_LO_CVT)  // A/B build: the explicit conversion
    uint32_t l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
    return l;
#else
    return __float_as_uint(r) + 0x1000u;
#endif
}

struct TileRaster {
    int tiles_m, tiles_n;
    __device__ void at(int t, int& tm, int& tn) const {
        const int group = t / (GROUP_M * tiles_n);
        const int first_m = group * GROUP_M;
        const int gsize = min(tiles_m - first_m, GROUP_M);
        tm = first_m + (t % (GROUP_M * tiles_n)) % gsize;
        tn = (t % (GROUP_M * tiles_n)) / gsize;
    }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b, int M,
                       int N, int K, float alpha, float beta, float* __restrict__ C, long long ldc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* conv = full + STAGES;
    uint64_t* empty = conv + STAGES;
    uint64_t* tmem_full = empty + STAGES;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint32_t* tmem_slot = (uint32_t*)(tmem_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    const TileRaster ras{(M + TILE_M - 1) / TILE_M, (N + TILE_N - 1) / TILE_N};
    const int ntiles = ras.tiles_m * ras.tiles_n;
    const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
    const int nk = (K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&conv[s], 2 * 4);  // 4 converter warps in each CTA
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tmem_full[b], 1);
            mbar_init(&tmem_empty[b], 2 * 4);  // 4 epilogue warps in each CTA
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_a) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_b) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync_all();  // barrier inits and the TMEM allocation visible to the peer CTA
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            int g = 0;
            for (int t = cluster; t < ntiles; t += nclusters) {
                int tm, tn;
                ras.at(t, tm, tn);
                const int m0 = tm * TILE_M + (int)rank * CTA_M;
                const int nb = tn * TILE_N + (int)rank * CTA_N;
                for (int kb = 0; kb < nk; kb++, g++) {
                    const int s = g % STAGES;
                    mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
                    uint8_t* st = smem + s * STAGE_BYTES;
                    mbar_expect_tx(&full[s], HI_BYTES);
                    tma_load_2d(st, &tm_a, &full[s], kb * BK, m0);
#pragma unroll
                    for (int c = 0; c < CTA_N / B_CHUNK; c++)
                        tma_load_2d(st + A_BYTES + c * B_CHUNK_BYTES, &tm_b, &full[s], nb + c * B_CHUNK, kb * BK);
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0 && lane == 0) {  // MMA issuer (leader CTA)
            int g = 0, i = 0;
            for (int t = cluster; t < ntiles; t += nclusters, i++) {
                const int b = i & 1;
                mbar_wait(&tmem_empty[b], ((i >> 1) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t d = tmem + (uint32_t)(b * TILE_N);
                for (int kb = 0; kb < nk; kb++, g++) {
                    const int s = g % STAGES;
                    mbar_wait(&conv[s], (g / STAGES) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
                    const uint64_t ahi = desc_a(sa), bhi = desc_b(sa + A_BYTES);
                    const uint64_t alo = desc_a(sa + HI_BYTES), blo = desc_b(sa + HI_BYTES + A_BYTES);
#pragma unroll
                    for (int ks = 0; ks < BK / 8; ks++) {
                        const uint64_t oa = (uint64_t)(ks * 32) >> 4;    // 8 tf32 = 32 B along K in the A atom
                        const uint64_t ob = (uint64_t)(ks * 1024) >> 4;  // 8 k = two 4-k atoms of B
                        const uint32_t acc = (kb | ks) != 0;
                        mma_tf32_2sm(d, alo + oa, bhi + ob, acc);  // small terms first
                        mma_tf32_2sm(d, ahi + oa, blo + ob, 1);
                        mma_tf32_2sm(d, ahi + oa, bhi + ob, 1);
                    }
                    commit_2sm(&empty[s]);  // frees the stage in both CTAs once these MMAs have read it
                }
                commit_2sm(&tmem_full[b]);
            }
        }
    } else if (warp < EPI_WARP0) {  // converters
        const int ct = threadIdx.x - 32 * CONV_WARP0;  // 0..127
        int g = 0;
        for (int t = cluster; t < ntiles; t += nclusters) {
            for (int kb = 0; kb < nk; kb++, g++) {
                const int s = g % STAGES;
                mbar_wait(&full[s], (g / STAGES) & 1);
                const uint32_t src = smem_u32(smem + s * STAGE_BYTES) + 16 * ct;
                uint4 v[HI_BYTES / 16 / 128];
#pragma unroll
                for (int j = 0; j < HI_BYTES / 16 / 128; j++) v[j] = lds128(src + j * 2048);
#pragma unroll
                for (int j = 0; j < HI_BYTES / 16 / 128; j++)
                    sts128(src + HI_BYTES + j * 2048,
                           make_uint4(lo_tf32(v[j].x), lo_tf32(v[j].y), lo_tf32(v[j].z), lo_tf32(v[j].w)));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(&conv[s]);
            }
        }
    } else {  // epilogue
        const int q = warp & 3;
        int i = 0;
        for (int t = cluster; t < ntiles; t += nclusters, i++) {
            int tm, tn;
            ras.at(t, tm, tn);
            const int b = i & 1;
            mbar_wait(&tmem_full[b], (i >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const int row = tm * TILE_M + (int)rank * CTA_M + q * 32 + lane;
            const int n0 = tn * TILE_N;
            for (int c0 = 0; c0 < TILE_N; c0 += 32) {
                uint32_t r[32];
                const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TILE_N + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                    "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                      "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
                      "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
                      "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
                      "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                if (row < M && n0 + c0 < N) {
                    float* crow = C + (long long)row * ldc + n0 + c0;
                    const int ncols = min(32, N - (n0 + c0));
                    if (ncols == 32 && ((uintptr_t)crow & 15) == 0) {
#pragma unroll
                        for (int v = 0; v < 8; v++) {
                            float4 o;
                            // C is read even when beta == 0: the fixture computes beta * C as written
                            // (0 * NaN / Inf in C is NaN, as in the emitted C)
                            const float4 old = *reinterpret_cast<const float4*>(crow + 4 * v);
                            o.x = alpha * __uint_as_float(r[4 * v + 0]) + beta * old.x;
                            o.y = alpha * __uint_as_float(r[4 * v + 1]) + beta * old.y;
                            o.z = alpha * __uint_as_float(r[4 * v + 2]) + beta * old.z;
                            o.w = alpha * __uint_as_float(r[4 * v + 3]) + beta * old.w;
                            *reinterpret_cast<float4*>(crow + 4 * v) = o;
                        }
                    } else {
#pragma unroll
                        for (int v = 0; v < 32; v++)
                            if (v < ncols)
                                crow[v] = alpha * __uint_as_float(r[v]) + beta * crow[v];
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&tmem_empty[b]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncwarp();        // producer / issuer lanes rejoin their warps before the aligned barrier
    cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
    }
}

// rows x cols (pitch spitch) -> dst with pitch dpitch (a multiple of 4 floats); the padding columns
// are never read (the tensor map's extent is cols)
__global__ void pack_rows_kernel(const float* __restrict__ src, long long spitch, long long rows, int cols,
                                 int dpitch, float* __restrict__ dst) {
    const long long total = rows * cols;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols, c = i - r * cols;
        dst[r * dpitch + c] = src[r * spitch + c];
    }
}

__global__ void scale_c_kernel(long long rows, int cols, long long ldc, float alpha, float beta,
                               float* __restrict__ C) {
    const long long n = rows * cols;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long r = i / cols;
        float* c = C + r * ldc + (i - r * cols);
        *c = alpha * 0.f + beta * *c;
    }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 2-D fp32 tensor map: inner extent `inner`, `outer` rows of `pitch` floats, box inner x outer
bool make_map(CUtensorMap* m, const float* base, int inner, int outer, long long pitch, int box_inner,
              int box_outer, CUtensorMapSwizzle sw) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// an operand TMA can read in place: 16-byte aligned base and row pitch
bool in_place(const void* p, long long pitch) { return ((uintptr_t)p & 15) == 0 && pitch % 4 == 0; }
size_t pad4(int c) { return ((size_t)c + 3) & ~(size_t)3; }

}  // namespace

size_t gemm_workspace_bytes(int m, int n, int k, const float* A, long long lda, const float* B, long long ldb) {
    size_t b = 0;
    if (!in_place(A, lda)) b += (size_t)m * pad4(k) * sizeof(float) + 256;
    if (!in_place(B, ldb)) b += (size_t)k * pad4(n) * sizeof(float) + 256;
    return b;
}

// C (m x n, row pitch ldc) = alpha A B + beta C with A m x k (pitch lda), B k x n (pitch ldb): the
// fixture's contiguous call has lda = k, ldb = n, ldc = n; strided views (a tile of a larger C, a
// column panel of B) pass their parents' pitches.
int launch_gemm(cudaStream_t st, int m, int n, int k, float alpha, float beta, const float* A, long long lda,
                const float* B, long long ldb, float* C, long long ldc, void* workspace, size_t workspace_bytes) {
    if (m <= 0 || n <= 0) return 0;
    if (lda < k || ldb < n || ldc < n) return (int)cudaErrorInvalidValue;
    if (workspace_bytes < gemm_workspace_bytes(m, n, k, A, lda, B, ldb)) return (int)cudaErrorInvalidValue;
    if (k == 0) {  // empty sum: C = alpha * 0 + beta * C, as the epilogue would write it
        scale_c_kernel<<<PENCIL_NUM_SMS * 8, 256, 0, st>>>(m, n, ldc, alpha, beta, C);
        return (int)cudaGetLastError();
    }
    uintptr_t ws = ((uintptr_t)workspace + 255) & ~(uintptr_t)255;
    const int grid_pack = PENCIL_NUM_SMS * 8;
    if (!in_place(A, lda)) {
        float* a2 = (float*)ws;
        const long long p = (long long)pad4(k);
        pack_rows_kernel<<<grid_pack, 256, 0, st>>>(A, lda, m, k, (int)p, a2);
        A = a2;
        lda = p;
        ws = ((uintptr_t)(a2 + (size_t)m * p) + 255) & ~(uintptr_t)255;
    }
    if (!in_place(B, ldb)) {
        float* b2 = (float*)ws;
        const long long p = (long long)pad4(n);
        pack_rows_kernel<<<grid_pack, 256, 0, st>>>(B, ldb, k, n, (int)p, b2);
        B = b2;
        ldb = p;
    }
    CUtensorMap maps[2];
    if (!make_map(&maps[0], A, k, m, lda, BK, CTA_M, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_map(&maps[1], B, n, k, ldb, B_CHUNK, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
        return (int)cudaErrorInvalidValue;
    static int max_clusters = 0;  // CTA pairs resident at once (one per two SMs)
    if (!max_clusters) {
        cudaFuncSetAttribute(gemm_3xtf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(PENCIL_NUM_SMS);
        cfg.blockDim = dim3(GEMM_THREADS);
        cfg.dynamicSmemBytes = SMEM_BYTES;
        int nc = 0;
        max_clusters = cudaOccupancyMaxActiveClusters(&nc, gemm_3xtf32_kernel, &cfg) == cudaSuccess && nc > 0
                           ? nc : PENCIL_NUM_SMS / 2;
        cudaGetLastError();
    }
    const int tiles = ((m + TILE_M - 1) / TILE_M) * ((n + TILE_N - 1) / TILE_N);
    const int clusters = tiles < max_clusters ? tiles : max_clusters;
    gemm_3xtf32_kernel<<<2 * clusters, GEMM_THREADS, SMEM_BYTES, st>>>(maps[0], maps[1], m, n, k, alpha, beta, C,
                                                                       ldc);
    return (int)cudaGetLastError();
}
