// CSR SpMV for the spmv.pencil.c nests (spmv_vec / spmv_inline / ACCESS-summarised spmv).
//
//   for (i = 0; i < nrows; i++) { s = 0; for (k = rowptr[i]; k < rowptr[i+1]; k++) s += val[k]*x[col[k]]; y[i] = s; }
//
// Inspector (plan): the nnz stream is cut into windows of TILE_NNZ non-zeros; tile t owns
// the rows whose first non-zero falls in window t (tile_row[t] = first row with
// rowptr[row] - rowptr[0] >= t*TILE_NNZ).  Built once per matrix by one pass over rowptr
// (csr_plan_kernel), it gives every warp a contiguous row range holding ~TILE_NNZ
// non-zeros regardless of the power-law row-length distribution.
//
// Executors (launch_csr_spmv picks one):
//   csr_seg_kernel — the default (16-byte-aligned col / val, monotone rowptr): per-lane segments over
//     the plan's row-start bitmap; rows scanned across lanes when reassociation is licensed
//     (spmv_vec), carried lane to lane in source order otherwise (spmv_inline, spmv); matrices with
//     empty rows name their rows through the plan's ordinals (EMPTY form).
//   csr_flow_kernel — the round-1 executor, now the A/B reference (-DPENCIL_VARIANT_NO_SEG) and the
//     entry that diverts a non-monotone rowptr to the generic schedule: the tile's non-zeros stream
//     in continuous 16-byte-per-lane windows and every 32-row batch is folded from whichever window
//     holds it (each lane its own row, in source order).
//   csr_stream_kernel — scalar loads, any alignment, same batch-and-fold structure.
// Every executor keeps the emitted C's rounding where source order is the contract: each product
// rounds on its own and each row sum is one chain of rounded adds, so spmv_inline and spmv (whose
// row loop is UNKNOWN, i.e. must stay sequential) are bit-identical to the reference-emitted C;
// spmv_vec's reduction pragma (PARALLEL_WITH_REDUCTION) licenses reassociation.
//
// Faults (E-INTERP analogues): col outside [0, ncols) or rowptr outside [0, nnz] set a bit
// in the status word and contribute 0.  A non-monotone rowptr (legal in PENCIL: the row
// is empty) switches the launch to a generic thread-per-row schedule.
#include "common.cuh"
#include "kernels.h"

#define SPMV_THREADS 256
// Plan windows: csr_tile_schedule (end of file).  Round 1's batch-and-fold executor swept
// {256..2048} x WCHUNK {64,128,256} at 2^24 rows (tools/spmv_sweep.sh): 1024 x 128 was its best
// (1.28 ms; 512: 1.34; 256: 1.59); the segmented executor runs 4096-non-zero windows.
// Non-zeros per lane per window and CTAs per SM of the segmented executor, per mode (2^24 rows,
// tools/ab_spmv_modes.sh): reassociated E 4 at 5 CTAs/SM (48 registers: the one-deep window
// pipeline) 1.137 ms, E 8 at 4 1.188; source order E 8 at 4 CTAs/SM 1.256 ms, E 4 at 5 1.302
// (its shuffle rounds are per window: wider windows halve them per non-zero), E 8 at 3 1.323.
#ifndef SEG_E
#define SEG_E 4
#endif
#ifndef SEG_CTAS_PER_SM
#define SEG_CTAS_PER_SM 5
#endif
#ifndef SEG_E_ORD
#define SEG_E_ORD 8
#endif
#ifndef SEG_CTAS_PER_SM_ORD
#define SEG_CTAS_PER_SM_ORD 4
#endif
#ifndef SEG_LANE0_MAX_E
#define SEG_LANE0_MAX_E 4  // widest window folded by lane 0 when it lies inside one row: at E 8 the
#endif                     // 256-add chain in one lane measured 1.310 ms against 1.257 with the rounds

// plan_flags: [0] non-monotone rowptr (generic schedule), [2] some row is empty.  rs_bits (when
// given): bit k set iff non-zero k is the first of its row — the row-start map of the segmented
// executor (csr_seg_kernel).
__global__ void csr_plan_kernel(int nrows, int nnz_len, const int* __restrict__ rowptr, TileSchedule ts,
                                int* __restrict__ tile_row, unsigned* __restrict__ plan_flags,
                                unsigned* __restrict__ rs_bits, unsigned* __restrict__ status) {
    const int base = __ldg(rowptr);
    const long long kA = ts.tail_start / ts.tile_nnz;  // tiles before the tapered tail
    // window k starts at B(k) = k T (k <= kA), tail_start + (k - kA) T2 after: first k with B(k) > o,
    // and last k with B(k) <= o
    auto first_above = [&](long long o) {
        return o < ts.tail_start ? o / ts.tile_nnz + 1 : kA + (o - ts.tail_start) / ts.tail_nnz + 1;
    };
    auto last_at_or_below = [&](long long o) {
        return o < ts.tail_start ? o / ts.tile_nnz : kA + (o - ts.tail_start) / ts.tail_nnz;
    };
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= nrows;
         i += (long long)gridDim.x * blockDim.x) {
        const int raw = __ldg(rowptr + i);
        if (raw < 0 || raw > nnz_len) raise_fault(status, FAULT_BAD_ROWPTR);
        const long long cur = (long long)raw - base;
        long long prev = -1;
        if (i > 0) {
            const int praw = __ldg(rowptr + i - 1);
            prev = (long long)praw - base;
            if (cur < prev) atomicOr(plan_flags, 1u);  // non-monotone -> generic schedule
            if (cur == prev) atomicOr(plan_flags + 2, 1u);  // row i - 1 is empty
            if (rs_bits && cur > prev && praw >= 0 && praw < nnz_len)
                atomicOr(rs_bits + (praw >> 5), 1u << (praw & 31));
        }
        if (cur <= prev) continue;
        long long k_lo = prev < 0 ? 0 : first_above(prev);
        long long k_hi = last_at_or_below(cur);
        if (k_hi > ts.ntiles - 1) k_hi = ts.ntiles - 1;
        for (long long k = k_lo; k <= k_hi; k++) tile_row[k] = (int)i;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tile_row[ts.ntiles] = nrows;
}

// Row result store.  DIST (fused SpMV -> all-gather, launch_csr_spmv_dist): the value also goes
// to every peer's copy of the gathered vector — one multimem store when an NVLS multicast
// address is given (the switch replicates it to all ranks), else one store per peer mapping.
// Row results of a warp are consecutive, so either form leaves as 128-byte NVLink writes.
template <bool DIST, bool LOCAL = true>
__device__ __forceinline__ void put_row(float* __restrict__ y, const PeerSet& ps, long long row, float s) {
    if (LOCAL) y[row] = s;
    if (DIST) {
        if (ps.mc)
            asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(ps.mc + row), "f"(s) : "memory");
        else
#pragma unroll
            for (int q = 0; q < PENCIL_MAX_PEERS; q++)  // unrolled: no local-memory copy of the params
                if (q < ps.n) ps.p[q][row] = s;
    }
}

// Generic schedule (any rowptr): one thread per row, loads straight from global.
template <bool DIST>
__device__ void spmv_generic_t(int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr,
                               const int* __restrict__ col, const float* __restrict__ val,
                               const float* __restrict__ x, float* __restrict__ y,
                               unsigned* __restrict__ status, const PeerSet& ps) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
         i += (long long)gridDim.x * blockDim.x) {
        int lo = __ldg(rowptr + i), hi = __ldg(rowptr + i + 1);
        float s = 0.f;
        for (int k = lo; k < hi; k++) {
            if (k < 0 || k >= nnz_len) { raise_fault(status, FAULT_OOB_LOAD); break; }
            int c = __ldg(col + k);
            float xv = 0.f;
            if ((unsigned)c < (unsigned)ncols) xv = __ldg(x + c);
            else raise_fault(status, FAULT_OOB_LOAD);
            s = __fadd_rn(s, __fmul_rn(__ldg(val + k), xv));
        }
        put_row<DIST>(y, ps, i, s);
    }
}

__device__ void spmv_generic(int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr,
                             const int* __restrict__ col, const float* __restrict__ val,
                             const float* __restrict__ x, float* __restrict__ y,
                             unsigned* __restrict__ status) {
    spmv_generic_t<false>(nrows, ncols, nnz_len, rowptr, col, val, x, y, status, PeerSet{});
}

// Persistent warps, no CTA-wide barrier: the kernel is bound by the L1TEX rate of random
// 4-byte gathers (~1 per SM clock, tools/microbench.py), so what matters is that every warp
// keeps its gathers in flight independently of the others.  Each warp draws tiles from a
// ticket counter (so a warp stuck on a 4096-long row never idles a whole CTA).  Per batch of
// 32 rows (one row per lane) the warp streams the batch's non-zeros in chunks of WCHUNK:
// coalesced col/val loads and x gathers, products staged in the warp's own smem slice, then
// every lane folds its row's slice in source order.  With the reduction licensed (ASSOC),
// slices longer than 16 are folded by the whole warp instead (strided partials + tree).
#define WARPS_PER_CTA (SPMV_THREADS / 32)
#define WCHUNK 128
#define CTAS_PER_SM 8
// Skewed staging index: lane i folds row i, whose slice starts near i*len; without the skew
// rows of equal length 16 put 16 lanes on one bank (a 16-way conflict on every read).
__device__ __forceinline__ int skew(int t) { return t + (t >> 5); }
// the same pad, 4 floats per 32: 16-byte aligned slots for vector stores, conflict-free reads
__device__ __forceinline__ int skew4(int t) { return t + 4 * (t >> 5); }

// Fold of one staged window into the lanes' rows: lane r adds the products of its row that lie in
// [lo, hi) (window positions, `base` = the window's first position).  Source order: each lane
// adds its slice in order, product-then-sum rounding as the emitted C.  With the reduction
// licensed (ASSOC), slices longer than 16 are folded by the whole warp instead (strided
// partials + shuffle tree), one such row at a time.  IDX maps a window offset to its skewed
// staging slot.
// in-order sum of staged products [lo, hi): U loads issued ahead of their adds (the adds stay
// in source order; only the smem latency is overlapped).  Source-order mode (U = 4): 1.567 ->
// 1.536 ms at 2^24 rows and no spills; with the reduction licensed the short slices it sees are
// better off plain (U = 4 / 8 there: 1.251 -> 1.283 / 1.271 ms).
template <int (*IDX)(int), int U>
__device__ __forceinline__ float fold_serial(float s, int lo, int hi, int base, const float* sp) {
    int t = lo;
    if (U > 1) {
        for (; t + U <= hi; t += U) {
            float v[U];
#pragma unroll
            for (int k = 0; k < U; k++) v[k] = sp[IDX(t + k - base)];
#pragma unroll
            for (int k = 0; k < U; k++) s = __fadd_rn(s, v[k]);
        }
    }
    for (; t < hi; t++) s = __fadd_rn(s, sp[IDX(t - base)]);
    return s;
}

template <bool ASSOC, int (*IDX)(int)>
__device__ __forceinline__ float fold_window(float s, int lo, int hi, int base, const float* sp, int lane) {
    if (ASSOC) {
        unsigned big = __ballot_sync(0xffffffffu, hi - lo > 16);
        if (hi - lo <= 16) s = fold_serial<IDX, 1>(s, lo, hi, base, sp);
        while (big) {
            const int o = __ffs(big) - 1;
            big &= big - 1;
            const int olo = __shfl_sync(0xffffffffu, lo, o), ohi = __shfl_sync(0xffffffffu, hi, o);
            float part = 0.f;
            for (int t = olo + lane; t < ohi; t += 32) part += sp[IDX(t - base)];
            part = warp_sum<32>(part);
            if (lane == o) s += part;
        }
    } else {
        s = fold_serial<IDX, 4>(s, lo, hi, base, sp);
    }
    return s;
}

template <bool ASSOC, int WCH>
__global__ void __launch_bounds__(SPMV_THREADS, CTAS_PER_SM) csr_stream_kernel(
    int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr, const int* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ x, float* __restrict__ y,
    const int* __restrict__ tile_row, int ntiles, const unsigned* __restrict__ plan,
    unsigned* __restrict__ tk, unsigned* __restrict__ status) {
    __shared__ float s_prod[WARPS_PER_CTA][WCH + WCH / 32];
    if (plan[0]) {  // non-monotone rowptr, flagged by the plan kernel earlier on this stream
        spmv_generic(nrows, ncols, nnz_len, rowptr, col, val, x, y, status);
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned total_warps = gridDim.x * WARPS_PER_CTA;
    float* sp = s_prod[warp];
    for (;;) {
    unsigned ticket = 0;
    if (lane == 0) ticket = atomicAdd(tk, 1u);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket >= (unsigned)ntiles) {
        // every warp draws exactly one failing ticket; the last one re-arms the counter
        if (lane == 0 && ticket == (unsigned)ntiles + total_warps - 1) *tk = 0;
        return;
    }
    const int tile = (int)ticket;
    const int r0 = __ldg(tile_row + tile), r1 = __ldg(tile_row + tile + 1);
    for (int rb = r0; rb < r1; rb += 32) {
        const int re = min(rb + 32, r1);
        const int row = rb + lane;
        const bool active = row < re;
        int my_s = 0, my_e = 0;
        if (active) {
            my_s = __ldg(rowptr + row);
            my_e = __ldg(rowptr + row + 1);
        }
        const int q_begin = max(__shfl_sync(0xffffffffu, my_s, 0), 0);
        const int q_end = min(__ldg(rowptr + re), nnz_len);
        float s = 0.f;
        for (int q = q_begin; q < q_end; q += WCH) {
            const int cnt = min(WCH, q_end - q);
            int c[WCH / 32];
            float v[WCH / 32], xv[WCH / 32];
#pragma unroll
            for (int u = 0; u < WCH / 32; u++) {
                const int t = u * 32 + lane;
                c[u] = t < cnt ? ld_stream_i(col + q + t) : 0;
                v[u] = t < cnt ? ld_stream_f(val + q + t) : 0.f;
            }
#pragma unroll
            for (int u = 0; u < WCH / 32; u++) {
                xv[u] = 0.f;
                if (u * 32 + lane < cnt) {
                    if ((unsigned)c[u] < (unsigned)ncols) xv[u] = ld_gather_f(x + c[u]);
                    else raise_fault(status, FAULT_OOB_LOAD);
                }
            }
#pragma unroll
            for (int u = 0; u < WCH / 32; u++)  // the product rounds on its own (emitted C as written)
                sp[skew(u * 32 + lane)] = __fmul_rn(v[u], xv[u]);
            __syncwarp();
            const int lo = max(my_s, q), hi = min(my_e, q + cnt);
            s = fold_window<ASSOC, skew>(s, lo, hi, q, sp, lane);
            __syncwarp();
        }
        if (active) y[row] = s;
    }
    }  // tickets
}

// Continuous-stream executor: the tile's non-zeros are streamed in
// full 4-aligned 128-element windows from its first to its last non-zero, independent of the
// 32-row batches, and every batch overlapping a window is folded from it (a batch that ends
// inside a window writes y and the next batch — prefetched — continues in the same window).
// The batch-aligned kernel restarts its windows at every batch, so each 32-row batch (~512
// non-zeros here) pays a partial first and last window.
// Measured and dropped (2^24 rows, A/B on one box): drawing the next tile's ticket one tile ahead
// (settled after the first window, two extra registers): 1.288 vs 1.239 ms; and, as a bound on
// the fold's cost, the same kernel with the fold replaced by one shared load per batch (wrong
// results): 1.292 ms — neither the tile-start round trips nor the fold is what separates this
// kernel from the 1.01 ms row-free gather stream; both edits cost the gather loop its schedule.
// Source order (spmv_inline): a long row's serial fold holds its warp's gathers (rows > 32 / 64 /
// 128 left unfolded, wrong results: 1.21 / 1.25 / 1.30 ms vs 1.52), but deferring them — products
// parked in a plan scratch (nnz floats) by the flow kernel, folded in order by a second,
// warp-per-row pass — measured 1.69 / 1.60 ms at thresholds 64 / 128: the scratch stream and the
// extra code in the window loop cost more than the freed gathers gain.  Dropped.
// DIST: fused SpMV -> all-gather (put_row); the warp fences its peer stores at system scope
// before it retires, so the barrier that follows the launch publishes them.
template <bool ASSOC, bool DIST = false>
__global__ void __launch_bounds__(SPMV_THREADS, CTAS_PER_SM) csr_flow_kernel(
    int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr, const int* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ x, float* __restrict__ y,
    const int* __restrict__ tile_row, int ntiles, const unsigned* __restrict__ plan,
    unsigned* __restrict__ tk, unsigned* __restrict__ status, const PeerSet ps) {
    __shared__ __align__(16) float s_prod[WARPS_PER_CTA][128 + 16];
    if (plan[0]) {
        spmv_generic_t<DIST>(nrows, ncols, nnz_len, rowptr, col, val, x, y, status, ps);
        if (DIST) __threadfence_system();
        return;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned total_warps = gridDim.x * WARPS_PER_CTA;
    float* sp = s_prod[warp];
    auto clampp = [&](int v) { return v < 0 ? 0 : (v > nnz_len ? nnz_len : v); };
    for (;;) {
        unsigned ticket = 0;
        if (lane == 0) ticket = atomicAdd(tk, 1u);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket >= (unsigned)ntiles) {
            if (lane == 0 && ticket == (unsigned)ntiles + total_warps - 1) *tk = 0;
            if (DIST) __threadfence_system();
            return;
        }
        const int r0 = __ldg(tile_row + ticket), r1 = __ldg(tile_row + ticket + 1);
        if (r0 >= r1) continue;
        // batch state: rows [rb, rb + 32), lane = row rb + lane; s_l = start of row rb + lane
        int rb = r0;
        int s_l = __ldg(rowptr + min(rb + lane, r1)), e_b = __ldg(rowptr + min(rb + 32, r1));
        int n_s = 0, n_e = 0;  // the next batch, prefetched
        if (rb + 32 < r1) {
            n_s = __ldg(rowptr + min(rb + 32 + lane, r1));
            n_e = __ldg(rowptr + min(rb + 64, r1));
        }
        const int P0 = clampp(__shfl_sync(0xffffffffu, s_l, 0));
        const int P1 = max(P0, clampp(__ldg(rowptr + r1)));
        auto bounds = [&](int& my_s, int& my_e) {
            my_s = clampp(s_l);
            my_e = __shfl_down_sync(0xffffffffu, s_l, 1);
            if (lane == 31) my_e = e_b;
            my_e = max(my_s, clampp(my_e));
            if (rb + lane >= r1) my_s = my_e = 0;
        };
        int my_s, my_e;
        bounds(my_s, my_e);
        int bend = clampp(e_b);
        float s = 0.f;
        for (int qa = P0 & ~3; qa < P1; qa += 128) {
            const int p = qa + 4 * lane;
            float pr[4] = {0.f, 0.f, 0.f, 0.f};
            if (p + 3 >= P0 && p < P1) {
                int c[4];
                float v[4];
                if (p + 3 < nnz_len) {
                    const int4 c4 = ld_stream_i4(reinterpret_cast<const int4*>(col + p));
                    const float4 v4 = ld_stream_f4(reinterpret_cast<const float4*>(val + p));
                    c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
                    v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; k++) {
                        c[k] = p + k < nnz_len ? __ldg(col + p + k) : 0;
                        v[k] = p + k < nnz_len ? __ldg(val + p + k) : 0.f;
                    }
                }
                // the 4 gathers issue unconditionally (masked / out-of-range entries read x[0]), so
                // they leave back to back instead of one branch region each
                bool use[4];
                float xv[4];
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const bool in = p + k >= P0 && p + k < P1, ok = (unsigned)c[k] < (unsigned)ncols;
                    use[k] = in && ok;
                    xv[k] = ld_gather_f(x + (use[k] ? c[k] : 0));
                    if (in && !ok) raise_fault(status, FAULT_OOB_LOAD);
                }
#pragma unroll
                for (int k = 0; k < 4; k++) pr[k] = use[k] ? __fmul_rn(v[k], xv[k]) : 0.f;  // rounds on its own
            }
            *reinterpret_cast<float4*>(sp + skew4(4 * lane)) = make_float4(pr[0], pr[1], pr[2], pr[3]);
            __syncwarp();
            for (;;) {  // fold every batch overlapping this window
                const int lo = max(my_s, qa), hi = min(my_e, qa + 128);
                s = fold_window<ASSOC, skew4>(s, lo, hi, qa, sp, lane);
                if (bend > qa + 128 || rb >= r1) break;  // the batch continues in the next window
                if (rb + lane < r1) y[rb + lane] = s;      // batch complete
                s = 0.f;
                rb += 32;
                if (rb >= r1) break;
                s_l = n_s;
                e_b = n_e;
                if (rb + 32 < r1) {
                    n_s = __ldg(rowptr + min(rb + 32 + lane, r1));
                    n_e = __ldg(rowptr + min(rb + 64, r1));
                }
                bounds(my_s, my_e);
                bend = clampp(e_b);
            }
            __syncwarp();
        }
        while (rb < r1) {  // batches past the last non-zero (empty rows)
            if (rb + lane < r1) y[rb + lane] = s;
            s = 0.f;
            rb += 32;
            if (rb >= r1) break;
            s_l = n_s;
            e_b = n_e;
            if (rb + 32 < r1) {
                n_s = __ldg(rowptr + min(rb + 32 + lane, r1));
                n_e = __ldg(rowptr + min(rb + 64, r1));
            }
        }
        if (DIST) {
            // the tile's rows leave together after its fold loop, re-read from y (L2) two rows per
            // lane at a time.  Measured at 2^24 rows with 1 / 7 local targets: +56 / +178 us over
            // the plain SpMV; storing from registers at each batch instead costs +170 / +420 us
            // (the store code in the fold loop costs the gather loop its schedule)
            __syncwarp();
            for (int r = r0 + lane; r < r1; r += 64) {
                const float v0 = y[r], v1 = r + 32 < r1 ? y[r + 32] : 0.f;
                put_row<true, false>(y, ps, r, v0);
                if (r + 32 < r1) put_row<true, false>(y, ps, r + 32, v1);
            }
        }
    }
}

// Segmented-reduction executor (reassociation licensed: spmv_vec; rows never empty — the plan's
// flag — so the k-th row start after a tile's first row is row r0 + k).  The tile's non-zeros
// stream in 128-element windows as in csr_flow_kernel (16-byte col / val loads, 4 gathers per
// lane), but instead of staging products and folding each row in its own lane, every lane reduces
// its 4 products by segments (the row starts come from the plan's bitmap, one 32-bit word per
// lane) and a warp segmented scan (5 shuffle rounds) carries the open row across lanes and windows;
// every row is stored once, by the lane where it closes.  Windows strictly inside the tile take a
// mask-free path (warp-uniform branch); faults are OR-ed per lane over the tile and raised once.
// The sum order is fixed (lanes in order, the scan tree, windows in order): deterministic.
// Measured at 2^24 rows (tools/ab_spmv.sh, one box): 1.241 ms on csr_flow_kernel -> 1.166 with
// this executor (1024-nnz tiles) -> 1.145 with 4096-nnz tiles (2048: 1.148, 8192: 1.159); the
// row-free stream + gather probe on the same data runs 1.010 ms.  ncu: 359 M warp instructions
// (flow kernel 857 M), L1TEX 89.6% (probe 95%).  Timing-only ablations (wrong results, not
// kept): no scan 1.084, no y stores 1.124, no row-start words 1.126.  Tried and dropped: 8
// non-zeros per lane (1.16-1.19: fewer warps or spills), the next window's col / val loads issued
// before this window's gathers (no gain), a ballot-based segmented scan with one shuffle per
// round (1.160: more ALU), and L2 evict-first stores / row-start loads (no change).
struct SegState {
    int row;      // the row open at the next window's first position (its ordinal among the
                  // non-empty rows when the matrix has empty rows)
    float carry;  // its partial sum from the earlier windows
    bool bad;     // a column index outside [0, ncols) was seen
    const int* rowmap;  // plans with empty rows: ordinal -> row (NULL: ordinal == row)
};

__device__ __forceinline__ void seg_store(float* p, float v) { __stcs(p, v); }
// y's element of the row with ordinal o
__device__ __forceinline__ float* seg_addr(float* y, const SegState& S, int o) {
    return y + (S.rowmap ? __ldg(S.rowmap + o) : o);
}

// Row starts in the lanes before this one and in the whole window, from one ballot per bit of the
// lane's count (0 .. E): VOTE + POPC on the ALU instead of a five-round shuffle scan (MIO, which the
// gathers need).
template <int E>
__device__ __forceinline__ void seg_start_counts(int lane, int cnt, int& before, int& total) {
    constexpr int NB = E < 2 ? 1 : E < 4 ? 2 : E < 8 ? 3 : E < 16 ? 4 : 5;  // bits of cnt <= E
    const unsigned lt = (1u << lane) - 1u;
    before = 0;
    total = 0;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const unsigned m = __ballot_sync(0xffffffffu, (cnt >> b) & 1);
        before += __popc(m & lt) << b;
        total += __popc(m) << b;
    }
}

// Source order (spmv_inline, ACCESS spmv: the row loop must fold in order) on the same window: a
// row's sum is one chain s = (((0 + p_a) + p_b) + ...), each add rounded, so a row spanning several
// lanes is carried from lane to lane instead of scanned.  A lane holding a row start ("breaker")
// knows its outgoing carry at once (its tail, folded from 0); a lane without one needs the carry
// of the lane before it.  R rounds of (shuffle up, refold) settle every chain, R = the longest run
// of breaker-free lanes (ballot; ~4 for 16-nnz rows, 32 under a long row — the serial chain of
// the row itself, which source order cannot avoid).  Then each breaker folds its head onto the
// settled incoming carry and stores the row that closes there; rows wholly inside the lane fold
// from 0 and are stored in order.  Masked positions carry +0, and s + 0 == s for every s the
// chain can hold (it starts at +0, so it is never -0): bit-identical to the emitted C.
template <int E>
__device__ __forceinline__ void seg_ordered(int lane, unsigned sb, const float (&pr)[E], float* __restrict__ y,
                                            SegState& S, float* __restrict__ sfold) {
    const bool brk = sb != 0;
    const int f = brk ? __ffs(sb) - 1 : E, l = brk ? 31 - __clz(sb) : E;
    auto fold_all = [&](float c) {
#pragma unroll
        for (int k = 0; k < E; k++) c = __fadd_rn(c, pr[k]);
        return c;
    };
    float co;
    if (brk) {
        co = 0.f;
#pragma unroll
        for (int k = 0; k < E; k++)
            if (k >= l) co = __fadd_rn(co, pr[k]);
    } else {
        co = fold_all(lane == 0 ? S.carry : 0.f);
    }
    const unsigned nb = __ballot_sync(0xffffffffu, brk);
    if (E % 4 == 0 && E <= SEG_LANE0_MAX_E && nb == 0) {
        // the whole window continues one row (rows > 32 E non-zeros): its chain is 32 E adds in a
        // row whichever way it is split, so lane 0 folds the staged products itself — 8 E LDS.128 +
        // 32 E FADD instead of 32 shuffle-and-refold rounds
        float4* sf = reinterpret_cast<float4*>(sfold);
#pragma unroll
        for (int h = 0; h < E / 4; h++)
            sf[lane * (E / 4) + h] = make_float4(pr[4 * h], pr[4 * h + 1], pr[4 * h + 2], pr[4 * h + 3]);
        __syncwarp();
        float c = S.carry;
        if (lane == 0) {
#pragma unroll 8
            for (int q = 0; q < 8 * E; q++) {
                const float4 v = sf[q];
                c = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(c, v.x), v.y), v.z), v.w);
            }
        }
        S.carry = __shfl_sync(0xffffffffu, c, 0);
        __syncwarp();  // the slice is free for the next window
        return;
    }
    unsigned run = ~nb;
    int R = 0;
    while (run) {  // longest run of breaker-free lanes (warp-uniform)
        run &= run << 1;
        R++;
    }
    for (int r = 0; r < R; r++) {
        const float ci = __shfl_up_sync(0xffffffffu, co, 1);
        if (!brk && lane > 0) co = fold_all(ci);
    }
    float ci = __shfl_up_sync(0xffffffffu, co, 1);
    if (lane == 0) ci = S.carry;
    int before, total;  // row starts in the lanes before this one / in the window
    seg_start_counts<E>(lane, __popc(sb), before, total);
    if (brk) {  // rows closing here: the open one (head on the incoming carry), then the inner rows
        const int ro = S.row + before;
        float h = ci;
#pragma unroll
        for (int k = 0; k < E; k++)
            if (k < f) h = __fadd_rn(h, pr[k]);
        __stcs(seg_addr(y, S, ro), h);
        float a = 0.f;
        int nseg = 0;
#pragma unroll
        for (int k = 0; k < E; k++) {
            if (k < f || k >= l) continue;
            if (k > f && ((sb >> k) & 1u)) {
                __stcs(seg_addr(y, S, ro + 1 + nseg), a);
                a = 0.f;
                nseg++;
            }
            a = __fadd_rn(a, pr[k]);
        }
        if (l > f) __stcs(seg_addr(y, S, ro + 1 + nseg), a);  // the row from the last-but-one start closes at l
    }
    S.carry = __shfl_sync(0xffffffffu, co, 31);
    S.row += total;
}

// One window of E * 32 non-zeros (E per lane: E / 4 16-byte loads per array per lane, all E gathers
// in flight together), split in two halves so that the tile loop can issue window w+1's loads and
// gathers before it reduces window w (the reduction's shuffle rounds then overlap gathers in flight
// instead of leaving the warp without any).  FULL: every position inside the tile (no masks).
template <int E>
struct SegWin {
    float v[E], xv[E];
    unsigned use;  // bit k: position p + k is in the tile with a valid column
    unsigned sb;   // bit k: position p + k starts a row (other than the tile's first)
};

// The window's col / val / row-start loads (streaming) and its x gathers (issued unconditionally:
// masked / invalid entries read x[0], so the E gathers leave back to back).
template <int E, bool FULL>
__device__ __forceinline__ void seg_fetch(int qa, int P0, int P1, int nnz_len, int ncols, int lane,
                                          const int* __restrict__ col, const float* __restrict__ val,
                                          const float* __restrict__ x, const unsigned* __restrict__ rs_bits,
                                          SegWin<E>& w, bool& bad) {
    constexpr unsigned EMASK = (1u << E) - 1u;
    const int p = qa + E * lane;  // qa is E-aligned, so the lane's E row-start bits share a word
    w.use = 0;
    w.sb = 0;
#pragma unroll
    for (int k = 0; k < E; k++) w.v[k] = w.xv[k] = 0.f;
    if (FULL || (p + E - 1 >= P0 && p < P1)) {
        int c[E];
        if (FULL || p + E - 1 < nnz_len) {
#pragma unroll
            for (int h = 0; h < E / 4; h++) {
                const int4 c4 = ld_stream_i4(reinterpret_cast<const int4*>(col + p + 4 * h));
                const float4 v4 = ld_stream_f4(reinterpret_cast<const float4*>(val + p + 4 * h));
                c[4 * h] = c4.x; c[4 * h + 1] = c4.y; c[4 * h + 2] = c4.z; c[4 * h + 3] = c4.w;
                w.v[4 * h] = v4.x; w.v[4 * h + 1] = v4.y; w.v[4 * h + 2] = v4.z; w.v[4 * h + 3] = v4.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < E; k++) {
                c[k] = p + k < nnz_len ? __ldg(col + p + k) : 0;
                w.v[k] = p + k < nnz_len ? __ldg(val + p + k) : 0.f;
            }
        }
        // the row-start words stream (evict-first, 32 MB): x keeps the L2
        unsigned sb = (ld_stream_u(rs_bits + (p >> 5)) >> (p & 31)) & EMASK;
        unsigned use = 0;
#pragma unroll
        for (int k = 0; k < E; k++) {
            const bool in = FULL || (p + k >= P0 && p + k < P1), ok = (unsigned)c[k] < (unsigned)ncols;
            w.xv[k] = ld_gather_f(x + (in && ok ? c[k] : 0));
            use |= (unsigned)(in && ok) << k;
            bad |= in && !ok;
            if (!FULL && !(p + k > P0 && p + k < P1)) sb &= ~(1u << k);
        }
        w.use = use;
        w.sb = sb;
    }
}

template <int E, bool ORDERED>
__device__ __forceinline__ void seg_reduce(int lane, const SegWin<E>& w, float* __restrict__ y, SegState& S,
                                           float* __restrict__ sfold) {
    float pr[E];
#pragma unroll
    for (int k = 0; k < E; k++) pr[k] = (w.use >> k) & 1u ? __fmul_rn(w.v[k], w.xv[k]) : 0.f;  // rounds on its own
    const unsigned sb = w.sb;
    if (ORDERED) {
        seg_ordered<E>(lane, sb, pr, y, S, sfold);
        return;
    }
    // the lane's segments: head (before its first start: closes the row open on entry), tail (from
    // its last start: stays open); rows that begin and end inside the lane (cnt >= 2) are stored
    // after the scan
    const int cnt = __popc(sb);
    const int f = sb ? __ffs(sb) - 1 : E, l = sb ? 31 - __clz(sb) : E;
    float head = f > 0 ? pr[0] : 0.f, acc = l <= 0 ? pr[0] : 0.f;
#pragma unroll
    for (int k = 1; k < E; k++) {
        head += f > k ? pr[k] : 0.f;
        acc += l <= k ? pr[k] : 0.f;
    }
    // one scan, two shuffles per round: the starts in lanes <= this one packed with the segment
    // flag, and the open row's partial sum, summed only while no start has been crossed (the
    // window carry enters at lane 0).  (Heads from one ballot with value-only shuffles, over the
    // rounds the window needs or all five, with the start counts from ballots: 1.163 ms against
    // 1.133 for this form at the same 48 registers — the per-lane head distance and ballot counts
    // cost more than the five flag shuffles here; the source-order path gains from them.)
    float sv = cnt ? acc : head + (lane == 0 ? S.carry : 0.f);
    int pk = (cnt << 1) | (cnt != 0);
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const float vo = __shfl_up_sync(0xffffffffu, sv, d);
        const int po = __shfl_up_sync(0xffffffffu, pk, d);
        if (lane >= d) {
            if (!(pk & 1)) sv = vo + sv;
            pk = (((pk >> 1) + (po >> 1)) << 1) | ((pk | po) & 1);
        }
    }
    const int win_starts = __shfl_sync(0xffffffffu, pk, 31) >> 1;
    const int before = (pk >> 1) - cnt;
    float excl = __shfl_up_sync(0xffffffffu, sv, 1);
    if (lane == 0) excl = S.carry;
    if (cnt) {  // y streams out (evict-first): its 64 MB must not push x out of L2
        const int ro = S.row + before;  // the row open on entry to this lane
        seg_store(seg_addr(y, S, ro), excl + head);
        if (cnt > 1) {  // rows wholly inside the lane
            float a = 0.f;
            int nseg = 0;
#pragma unroll
            for (int k = 0; k < E; k++) {
                if (k < f) continue;
                if (k > f && ((sb >> k) & 1u)) {
                    seg_store(seg_addr(y, S, ro + 1 + nseg), a);
                    a = 0.f;
                    nseg++;
                }
                if (nseg < cnt - 1) a += pr[k];
            }
        }
    }
    S.carry = __shfl_sync(0xffffffffu, sv, 31);
    S.row += win_starts;
}

// A tile's windows, software-pipelined one deep: window w+1's col / val / row-start loads and its
// gathers are issued before window w is reduced, so the reduction's shuffle rounds overlap gathers in
// flight.  Measured at 2^24 rows (tools/ab_spmv_modes.sh): vec / inline 1.145 / 1.306 ms unpipelined
// at 6 CTAs per SM -> 1.134 / 1.305 pipelined at 5 (at 6 the 40-register cap costs 1.19 / 1.32; at 4,
// 1.18 / 1.34).  Two deep (w+2's stream loads, w+1's gathers, w's reduction): 1.21 / 1.37 at 4 CTAs
// per SM and spills at 5 — the registers cost more warps than the deeper pipeline hides.  col / val
// staged through a per-warp shared-memory ring by bulk copies (lane 0, mbarrier completion, 2 / 4 / 5
// windows ahead) so that the gathers never wait for the column stream: 1.81-2.94 ms (same bits) —
// the per-warp 1 KB bulk copies are far slower than the LSU streams here.
template <int E, bool ORDERED>
__device__ __forceinline__ void seg_tile(int P0, int P1, int nnz_len, int ncols, int lane, const int* __restrict__ col,
                                         const float* __restrict__ val, const float* __restrict__ x,
                                         const unsigned* __restrict__ rs_bits, float* __restrict__ y, SegState& S,
                                         float* __restrict__ sfold) {
    constexpr int W = 32 * E;
    int qa = P0 & ~(E - 1);
    if (qa >= P1) return;
    SegWin<E> cur, nxt;
    // the first window always masks (positions before P0; P0's own start)
    seg_fetch<E, false>(qa, P0, P1, nnz_len, ncols, lane, col, val, x, rs_bits, cur, S.bad);
    for (;;) {
        const int qn = qa + W;
        const bool more = qn < P1;
        if (more) {
            if (qn + W <= P1) seg_fetch<E, true>(qn, P0, P1, nnz_len, ncols, lane, col, val, x, rs_bits, nxt, S.bad);
            else seg_fetch<E, false>(qn, P0, P1, nnz_len, ncols, lane, col, val, x, rs_bits, nxt, S.bad);
        }
        seg_reduce<E, ORDERED>(lane, cur, y, S, sfold);
        if (!more) break;
        cur = nxt;
        qa = qn;
    }
}

template <bool DIST, bool ORDERED, bool EMPTY>
__global__ void __launch_bounds__(SPMV_THREADS, ORDERED ? SEG_CTAS_PER_SM_ORD : SEG_CTAS_PER_SM) csr_seg_kernel(
    int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr, const int* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ x, float* __restrict__ y,
    const int* __restrict__ tile_row, int ntiles, const unsigned* __restrict__ plan,
    const unsigned* __restrict__ rs_bits, const int* __restrict__ ord, const int* __restrict__ rowmap,
    unsigned* __restrict__ tk, unsigned* __restrict__ status, const PeerSet ps) {
    if (plan[0]) {
        spmv_generic_t<DIST>(nrows, ncols, nnz_len, rowptr, col, val, x, y, status, ps);
        if (DIST) __threadfence_system();
        return;
    }
    const int lane = threadIdx.x & 31;
    const unsigned total_warps = gridDim.x * WARPS_PER_CTA;
    __shared__ __align__(16) float s_fold[ORDERED ? WARPS_PER_CTA : 1][ORDERED ? SEG_E_ORD * 32 : 4];  // a window
    float* sfold = s_fold[ORDERED ? threadIdx.x >> 5 : 0];
    auto clampp = [&](int v) { return v < 0 ? 0 : (v > nnz_len ? nnz_len : v); };
    for (;;) {
        unsigned ticket = 0;
        if (lane == 0) ticket = atomicAdd(tk, 1u);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        if (ticket >= (unsigned)ntiles) {
            if (lane == 0 && ticket == (unsigned)ntiles + total_warps - 1) *tk = 0;
            if (DIST) __threadfence_system();
            return;
        }
        const int r0 = __ldg(tile_row + ticket), r1 = __ldg(tile_row + ticket + 1);
        if (r0 >= r1) continue;
        const int P0 = clampp(__ldg(rowptr + r0));
        const int P1 = max(P0, clampp(__ldg(rowptr + r1)));
        if (P1 > P0) {  // (a tile of empty rows only has nothing to fold: their y is zeroed before the launch)
            // EMPTY is a compile-time flag so that without empty rows the row names fold to ordinals
            SegState S{EMPTY ? __ldg(ord + r0) : r0, 0.f, false, EMPTY ? rowmap : nullptr};
            seg_tile<ORDERED ? SEG_E_ORD : SEG_E, ORDERED>(P0, P1, nnz_len, ncols, lane, col, val, x, rs_bits, y, S,
                                                          sfold);
            if (lane == 0) seg_store(seg_addr(y, S, S.row), S.carry);  // the tile's last non-empty row
            if (S.bad) raise_fault(status, FAULT_OOB_LOAD);
        }
        if (DIST) {
            // the tile's rows leave together, re-read from y (L2) two per lane, as 128-byte runs.
            // Storing each row to the peers where it closes instead (one more scattered store per
            // row and peer) measured 1.427 ms against 1.274 for this at world 1 (one target).
            __syncwarp();
            for (int r = r0 + lane; r < r1; r += 64) {
                const float v0 = y[r], v1 = r + 32 < r1 ? y[r + 32] : 0.f;
                put_row<true, false>(y, ps, r, v0);
                if (r + 32 < r1) put_row<true, false>(y, ps, r + 32, v1);
            }
        }
    }
}

int launch_csr_plan(cudaStream_t st, int nrows, int nnz_len, const int* rowptr, const TileSchedule& ts,
                    int* tile_row, unsigned* plan_flags, unsigned* rs_bits, unsigned* status) {
    cudaMemsetAsync(plan_flags, 0, 64, st);  // [0] non-monotone flag, [2] empty-row flag
    if (rs_bits) cudaMemsetAsync(rs_bits, 0, csr_rs_words(nnz_len) * sizeof(unsigned), st);
    long long blocks = ((long long)nrows + 1 + 255) / 256;
    if (blocks > PENCIL_NUM_SMS * 16) blocks = PENCIL_NUM_SMS * 16;
    csr_plan_kernel<<<(int)blocks, 256, 0, st>>>(nrows, nnz_len, rowptr, ts, tile_row, plan_flags, rs_bits,
                                                 status);
    return (int)cudaGetLastError();
}

size_t csr_rs_words(int nnz_len) { return (size_t)(nnz_len > 0 ? nnz_len : 1) / 32 + 2; }

// Plans with empty rows (monotone rowptr): ord[r] = number of non-empty rows before row r
// (r = 0..nrows) and rowmap[ord[r]] = r for every non-empty row, so that the segmented executor
// — which counts row starts, i.e. non-empty rows — can name each row it closes.  Three passes of
// an exclusive scan over the rows: per-block counts, a one-block scan of those, and the per-block
// scans that write ord and rowmap.
constexpr int ORD_BLOCKS = 1024;
__device__ __forceinline__ int row_nonempty(const int* __restrict__ rowptr, long long r) {
    return __ldg(rowptr + r + 1) > __ldg(rowptr + r);
}
__global__ void csr_ord_count_kernel(int nrows, const int* __restrict__ rowptr, int* __restrict__ bsum) {
    const long long per = ((long long)nrows + ORD_BLOCKS - 1) / ORD_BLOCKS;
    const long long lo = blockIdx.x * per, hi = min((long long)nrows, lo + per);
    int c = 0;
    for (long long r = lo + threadIdx.x; r < hi; r += blockDim.x) c += row_nonempty(rowptr, r);
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ int ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)blockDim.x / 32; w++) t += ws[w];
        bsum[blockIdx.x] = t;
    }
}
__global__ void csr_ord_scan_blocks_kernel(int* __restrict__ bsum) {  // one block of ORD_BLOCKS threads
    __shared__ int s[ORD_BLOCKS];
    const int t = threadIdx.x;
    s[t] = bsum[t];
    __syncthreads();
    for (int d = 1; d < ORD_BLOCKS; d <<= 1) {  // inclusive Hillis-Steele
        const int v = t >= d ? s[t - d] : 0;
        __syncthreads();
        s[t] += v;
        __syncthreads();
    }
    bsum[t] = t ? s[t - 1] : 0;  // exclusive
}
__global__ void csr_ord_write_kernel(int nrows, const int* __restrict__ rowptr, const int* __restrict__ boff,
                                     int* __restrict__ ord, int* __restrict__ rowmap) {
    const long long per = ((long long)nrows + ORD_BLOCKS - 1) / ORD_BLOCKS;
    const long long lo = blockIdx.x * per, hi = min((long long)nrows, lo + per);
    __shared__ int ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int base = boff[blockIdx.x];
    for (long long r0 = lo; r0 < hi; r0 += blockDim.x) {
        const long long r = r0 + threadIdx.x;
        const int f = r < hi ? row_nonempty(rowptr, r) : 0;
        const unsigned b = __ballot_sync(0xffffffffu, f);
        if (lane == 0) ws[warp] = __popc(b);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < nw; w++) {
            before += w < warp ? ws[w] : 0;
            total += ws[w];
        }
        const int o = base + before + __popc(b & ((1u << lane) - 1u));
        if (r < hi) {
            ord[r] = o;
            if (f) rowmap[o] = (int)r;
        }
        base += total;
        __syncthreads();
    }
    if (hi == nrows && lo < hi && threadIdx.x == 0) ord[nrows] = base;
}

int launch_csr_ordinals(cudaStream_t st, int nrows, const int* rowptr, int* ord, int* rowmap, int* bsum) {
    if (nrows <= 0) return 0;
    csr_ord_count_kernel<<<ORD_BLOCKS, 256, 0, st>>>(nrows, rowptr, bsum);
    csr_ord_scan_blocks_kernel<<<1, ORD_BLOCKS, 0, st>>>(bsum);
    csr_ord_write_kernel<<<ORD_BLOCKS, 256, 0, st>>>(nrows, rowptr, bsum, ord, rowmap);
    return (int)cudaGetLastError();
}
size_t csr_ord_scratch_ints() { return ORD_BLOCKS; }

// the segmented executor's four forms (reassociated / source order, with / without empty rows)
template <bool DIST>
void seg_launch(cudaStream_t st, int grid, int assoc, int nrows, int ncols, int nnz_len, const int* rowptr,
                const int* col, const float* val, const float* x, float* y, const int* tile_row, int ntiles,
                const unsigned* plan_flags, const SegPlan& seg, unsigned* tk, unsigned* status, const PeerSet& ps) {
#define SEG_ARGS nrows, ncols, nnz_len, rowptr, col, val, x, y, tile_row, ntiles, plan_flags, seg.rs_bits, seg.ord, \
                 seg.rowmap, tk, status, ps
    if (seg.ord) {
        if (assoc) csr_seg_kernel<DIST, false, true><<<grid, SPMV_THREADS, 0, st>>>(SEG_ARGS);
        else csr_seg_kernel<DIST, true, true><<<grid, SPMV_THREADS, 0, st>>>(SEG_ARGS);
    } else {
        if (assoc) csr_seg_kernel<DIST, false, false><<<grid, SPMV_THREADS, 0, st>>>(SEG_ARGS);
        else csr_seg_kernel<DIST, true, false><<<grid, SPMV_THREADS, 0, st>>>(SEG_ARGS);
    }
#undef SEG_ARGS
}

// Executor choice: the continuous-stream kernel when col / val are 16-byte aligned (1.25 ms at
// 2^24 rows), else the scalar-load kernel (any alignment; 1.28 ms).  Measured and dropped (numbers
// at 2^24 rows; the code is in the git history before the round-2 clean-up, commit be69d3c):
//   * batch-aligned 128-bit kernel (windows restart at each 32-row batch): 1.265-1.273 ms; with 8
//     non-zeros per lane: 1.355 ms;
//   * TMA-fed col/val stream (per-warp 512-byte cp.async.bulk ring): 1.87 ms;
//   * 3-stage software-pipelined LSU variant: 1.41 ms (the chunk/batch merge doubled the
//     instruction count); cp.async double-buffered col/val prefetch: 2.43 ms (MIO-throttled);
//   * register prefetch of the next chunk's column indices: 1.34 ms at 8 CTAs/SM, 1.39 at 7;
//   * warp-specialised split (producer warps stream + gather into an mbarrier-handed smem ring,
//     one consumer warp per CTA folds): 1.89 ms with 3 producers per consumer, 2.73 with 7;
//   * cp.async.bulk.prefetch.L2 of the col/val windows 1 / 2 / 4 ahead: 1.38 / 1.45 / 1.41 ms;
//   * an L2 persisting access-policy window over x: DRAM read 4.30 -> 2.70 GB per SpMV but no
//     time gain (the request path, not DRAM, is the limit), and the set-aside L2 slowed the
//     caller's next streaming kernels 2.2-2.4x;
//   * window tile sizes 256 / 512 / 2048 non-zeros and chunks of 64 / 256: all slower than 1024 x 128.
// `tk` is the per-(device, stream) ticket word (runtime.cpp): the kernels draw tiles from it and
// the last warp re-arms it, so launches on one stream never share it with another stream's.
int launch_csr_spmv(cudaStream_t st, int assoc, int nrows, int ncols, int nnz_len,
                    const int* rowptr, const int* col, const float* val, const float* x, float* y,
                    const int* tile_row, int ntiles, const unsigned* plan_flags, const SegPlan& seg,
                    unsigned* tk, unsigned* status) {
    const unsigned* rs_bits = seg.rs_bits;
    if (nrows <= 0) return 0;
    int grid = (ntiles + WARPS_PER_CTA - 1) / WARPS_PER_CTA;  // persistent: at most one wave
    if (grid > PENCIL_NUM_SMS * CTAS_PER_SM) grid = PENCIL_NUM_SMS * CTAS_PER_SM;
    const bool aligned = (uintptr_t)col % 16 == 0 && (uintptr_t)val % 16 == 0;
#ifdef PENCIL_VARIANT_NO_SEG
    rs_bits = nullptr;  // A/B build: the batch-and-fold executor for every mode
#endif
    if (rs_bits && aligned) {  // segmented executor (scan, or carried in source order)
        const int cps = assoc ? SEG_CTAS_PER_SM : SEG_CTAS_PER_SM_ORD;
        if (grid > PENCIL_NUM_SMS * cps) grid = PENCIL_NUM_SMS * cps;
        seg_launch<false>(st, grid, assoc, nrows, ncols, nnz_len, rowptr, col, val, x, y, tile_row, ntiles, plan_flags,
                          seg, tk, status, PeerSet{});
        return (int)cudaGetLastError();
    }
    if (aligned) {
        if (assoc)
            csr_flow_kernel<true><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                 tile_row, ntiles, plan_flags, tk, status, PeerSet{});
        else
            csr_flow_kernel<false><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                  tile_row, ntiles, plan_flags, tk, status, PeerSet{});
    } else if (assoc) {
        csr_stream_kernel<true, WCHUNK><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                       tile_row, ntiles, plan_flags, tk, status);
    } else {
        csr_stream_kernel<false, WCHUNK><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                        tile_row, ntiles, plan_flags, tk, status);
    }
    return (int)cudaGetLastError();
}

// y rows -> peers (the distribution step on its own, for operands the fused kernel cannot take)
__global__ void dist_rows_kernel(int nrows, const float* __restrict__ y, const PeerSet ps) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
         i += (long long)gridDim.x * blockDim.x) {
        const float v = y[i];
        if (ps.mc)
            asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(ps.mc + i), "f"(v) : "memory");
        else
#pragma unroll
            for (int q = 0; q < PENCIL_MAX_PEERS; q++)
                if (q < ps.n) ps.p[q][i] = v;
    }
    __threadfence_system();
}

int launch_csr_spmv_dist(cudaStream_t st, int assoc, int nrows, int ncols, int nnz_len,
                         const int* rowptr, const int* col, const float* val, const float* x, float* y,
                         const int* tile_row, int ntiles, const unsigned* plan_flags, const SegPlan& seg,
                         unsigned* tk, unsigned* status, const PeerSet& peers) {
    const unsigned* rs_bits = seg.rs_bits;
    if (nrows <= 0) return 0;
    const bool aligned = (uintptr_t)col % 16 == 0 && (uintptr_t)val % 16 == 0;
    if (rs_bits && aligned) {
        int grid = (ntiles + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
        const int cps = assoc ? SEG_CTAS_PER_SM : SEG_CTAS_PER_SM_ORD;
        if (grid > PENCIL_NUM_SMS * cps) grid = PENCIL_NUM_SMS * cps;
        seg_launch<true>(st, grid, assoc, nrows, ncols, nnz_len, rowptr, col, val, x, y, tile_row, ntiles, plan_flags,
                         seg, tk, status, peers);
        return (int)cudaGetLastError();
    }
    if (aligned) {
        int grid = (ntiles + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
        if (grid > PENCIL_NUM_SMS * CTAS_PER_SM) grid = PENCIL_NUM_SMS * CTAS_PER_SM;
        if (assoc)
            csr_flow_kernel<true, true><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                       tile_row, ntiles, plan_flags, tk, status, peers);
        else
            csr_flow_kernel<false, true><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y,
                                                                        tile_row, ntiles, plan_flags, tk, status, peers);
        return (int)cudaGetLastError();
    }
    // unaligned col/val: the regular executor, then the rows leave in a second launch
    int e = launch_csr_spmv(st, assoc, nrows, ncols, nnz_len, rowptr, col, val, x, y, tile_row, ntiles,
                            plan_flags, SegPlan{}, tk, status);
    if (e) return e;
    long long blocks = ((long long)nrows + 255) / 256;
    if (blocks > PENCIL_NUM_SMS * 8) blocks = PENCIL_NUM_SMS * 8;
    dist_rows_kernel<<<(int)blocks, 256, 0, st>>>(nrows, y, peers);
    return (int)cudaGetLastError();
}

__global__ void csr_generic_kernel(int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr,
                                   const int* __restrict__ col, const float* __restrict__ val,
                                   const float* __restrict__ x, float* __restrict__ y,
                                   unsigned* __restrict__ status) {
    spmv_generic(nrows, ncols, nnz_len, rowptr, col, val, x, y, status);
}

int launch_csr_generic(cudaStream_t st, int nrows, int ncols, int nnz_len, const int* rowptr,
                       const int* col, const float* val, const float* x, float* y,
                       unsigned* status) {
    if (nrows <= 0) return 0;
    long long blocks = ((long long)nrows + 255) / 256;
    if (blocks > PENCIL_NUM_SMS * 16) blocks = PENCIL_NUM_SMS * 16;
    csr_generic_kernel<<<(int)blocks, 256, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val, x, y, status);
    return (int)cudaGetLastError();
}

// plan window per mode: source order (the batch-and-fold executor) and reassociated (segmented)
#ifndef SEG_TILE_NNZ
#define SEG_TILE_NNZ 8192
#endif
#ifndef SEG_TAIL_TILE_NNZ
#define SEG_TAIL_TILE_NNZ 1024  // 0: no tapered tail
#endif
#ifndef SEG_TAIL_WAVES
#define SEG_TAIL_WAVES 0.25  // tail length in full-size tiles per warp of the launch
#endif
// Tickets are drawn in matrix order, so the warps that draw the last full-size tiles start them
// up to one tile time before the end; the tail's smaller tiles (a quarter of a wave of the launch's
// warps of full-size tiles) keep the other warps busy meanwhile and end within a small tile of
// each other.
// Measured at 2^24 rows (tools/ab_spmv_modes.sh, two rounds): vec / inline 1.133 / 1.239 ms
// without the tail, 1.129 / 1.233 with it (1024-nnz tail tiles, 0.5 wave); 1 wave 1.132 / 1.234,
// 2 waves 1.139 / 1.238, 512-nnz tail tiles 1.141 / 1.241, 2048 1.132 / 1.234 — small: the
// request path is shared per SM, so an SM stays busy until its last few warps run dry.
// With the tail, larger full-size tiles pay (fewer tickets and window-pipeline restarts): 8192-nnz
// tiles with a quarter wave of 1024-nnz tail tiles (the same tail length) 1.110 / 1.215 ms against
// 1.116 / 1.224 for 4096 (16384: 1.112 / 1.219; 2048: 1.129 / 1.240; 2048-nnz tail tiles 1.113 / 1.218).
TileSchedule csr_tile_schedule(int mode, int nnz_len) {
    TileSchedule ts;
    const long long nnz = nnz_len > 0 ? nnz_len : 0;
    ts.tile_nnz = SEG_TILE_NNZ;
    ts.tail_nnz = SEG_TAIL_TILE_NNZ > 0 ? SEG_TAIL_TILE_NNZ : SEG_TILE_NNZ;
    const long long warps = (long long)PENCIL_NUM_SMS * (mode ? SEG_CTAS_PER_SM : SEG_CTAS_PER_SM_ORD) * WARPS_PER_CTA;
    long long tail = SEG_TAIL_TILE_NNZ > 0 ? (long long)(SEG_TAIL_WAVES * (double)warps * SEG_TILE_NNZ) : 0;
    // the tail starts on a full-size window boundary; small matrices are all tail or all full-size
    long long start = nnz - tail;
    start = start > 0 ? start / ts.tile_nnz * ts.tile_nnz : 0;
    ts.tail_start = start;
    const long long nt = start / ts.tile_nnz + (nnz - start + ts.tail_nnz - 1) / ts.tail_nnz;
    ts.ntiles = (int)(nt < 1 ? 1 : nt);
    return ts;
}
