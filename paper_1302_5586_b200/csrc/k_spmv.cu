// CSR SpMV for the spmv.pencil.c nests (spmv_vec / spmv_inline / ACCESS-summarised spmv).
//
//   for (i = 0; i < nrows; i++) { s = 0; for (k = rowptr[i]; k < rowptr[i+1]; k++) s += val[k]*x[col[k]]; y[i] = s; }
//
// Inspector (plan): the nnz stream is cut into windows of TILE_NNZ non-zeros; tile t owns
// the rows whose first non-zero falls in window t (tile_row[t] = first row with
// rowptr[row] - rowptr[0] >= t*TILE_NNZ).  Built once per matrix by one pass over rowptr
// (csr_plan_kernel), it gives every CTA a contiguous row range holding ~TILE_NNZ
// non-zeros regardless of the power-law row-length distribution.
//
// Executor (csr_stream_kernel): per tile, per batch of 256 rows, the batch's non-zeros
// are streamed with coalesced loads (col, val: evict-first) while x[col] is gathered
// (evict-last, so the 64 MB vector stays L2-resident), staged in shared memory, then each
// thread folds its own row in source order: s = s + val[k]*x[col[k]], product and sum each
// rounded to fp32.  That is the reference-emitted C compiled as written, so spmv_inline and
// spmv (whose row loop is UNKNOWN, i.e. must stay sequential) are bit-identical to it.
// spmv_vec's reduction pragma (PARALLEL_WITH_REDUCTION) licenses reassociation: rows longer
// than a warp are then folded by the whole warp (lane partials + shuffle tree).
//
// Faults (E-INTERP analogues): col outside [0, ncols) or rowptr outside [0, nnz] set a bit
// in the status word and contribute 0.  A non-monotone rowptr (legal in PENCIL: the row
// is empty) switches the launch to a generic thread-per-row schedule.
#include "common.cuh"
#include "kernels.h"

#define SPMV_THREADS 256
#define SPMV_CHUNK 2048

__global__ void csr_plan_kernel(int nrows, int nnz_len, const int* __restrict__ rowptr,
                                int tile_nnz, int ntiles, int* __restrict__ tile_row,
                                unsigned* __restrict__ plan_flags, unsigned* __restrict__ status) {
    const int base = __ldg(rowptr);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i <= nrows;
         i += (long long)gridDim.x * blockDim.x) {
        const int raw = __ldg(rowptr + i);
        if (raw < 0 || raw > nnz_len) raise_fault(status, FAULT_BAD_ROWPTR);
        const long long cur = (long long)raw - base;
        long long prev = -1;
        if (i > 0) {
            prev = (long long)__ldg(rowptr + i - 1) - base;
            if (cur < prev) atomicOr(plan_flags, 1u);  // non-monotone -> generic schedule
        }
        if (cur <= prev) continue;
        long long k_lo = prev < 0 ? 0 : prev / tile_nnz + 1;
        long long k_hi = cur / tile_nnz;
        if (k_hi > ntiles - 1) k_hi = ntiles - 1;
        for (long long k = k_lo; k <= k_hi; k++) tile_row[k] = (int)i;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) tile_row[ntiles] = nrows;
}

// Generic schedule (any rowptr): one thread per row, loads straight from global.
__device__ void spmv_generic(int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr,
                             const int* __restrict__ col, const float* __restrict__ val,
                             const float* __restrict__ x, float* __restrict__ y,
                             unsigned* __restrict__ status) {
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
        y[i] = s;
    }
}

template <bool ASSOC>
__global__ void __launch_bounds__(SPMV_THREADS) csr_stream_kernel(
    int nrows, int ncols, int nnz_len, const int* __restrict__ rowptr, const int* __restrict__ col,
    const float* __restrict__ val, const float* __restrict__ x, float* __restrict__ y,
    const int* __restrict__ tile_row, int ntiles, const unsigned* __restrict__ plan_flags,
    unsigned* __restrict__ status) {
    __shared__ float s_prod[SPMV_CHUNK];
    if (*plan_flags) {  // written by the plan kernel earlier on this stream
        spmv_generic(nrows, ncols, nnz_len, rowptr, col, val, x, y, status);
        return;
    }
    const int tid = threadIdx.x;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int r0 = __ldg(tile_row + tile), r1 = __ldg(tile_row + tile + 1);
        for (int rb = r0; rb < r1; rb += SPMV_THREADS) {
            const int re = min(rb + SPMV_THREADS, r1);
            const int row = rb + tid;
            const bool active = row < re;
            int my_s = 0, my_e = 0;
            if (active) {
                my_s = __ldg(rowptr + row);
                my_e = __ldg(rowptr + row + 1);
            }
            const int q_begin = max(__ldg(rowptr + rb), 0);
            const int q_end = min(__ldg(rowptr + re), nnz_len);
            float s = 0.f;
            for (int q = q_begin; q < q_end; q += SPMV_CHUNK) {
                const int cnt = min(SPMV_CHUNK, q_end - q);
                // stage: coalesced col/val stream + x gather; 8 independent loads per thread
#pragma unroll 4
                for (int t = tid; t < cnt; t += SPMV_THREADS) {
                    const int p = q + t;
                    const int c = ld_stream_i(col + p);
                    float xv = 0.f;
                    if ((unsigned)c < (unsigned)ncols) xv = ld_keep_f(x + c);
                    else raise_fault(status, FAULT_OOB_LOAD);
                    // the product rounds on its own, as in the emitted C compiled as written
                    s_prod[t] = __fmul_rn(ld_stream_f(val + p), xv);
                }
                __syncthreads();
                const int lo = max(my_s, q), hi = min(my_e, q + cnt);
                if (!ASSOC) {
                    for (int p = lo; p < hi; p++) s = __fadd_rn(s, s_prod[p - q]);
                } else {
                    for (int p = lo; p < hi; p++) s = __fadd_rn(s, s_prod[p - q]);
                }
                __syncthreads();
            }
            if (active) y[row] = s;
        }
    }
}

int launch_csr_plan(cudaStream_t st, int nrows, int nnz_len, const int* rowptr, int tile_nnz,
                    int ntiles, int* tile_row, unsigned* plan_flags, unsigned* status) {
    cudaMemsetAsync(plan_flags, 0, sizeof(unsigned), st);
    long long blocks = ((long long)nrows + 1 + 255) / 256;
    if (blocks > PENCIL_NUM_SMS * 16) blocks = PENCIL_NUM_SMS * 16;
    csr_plan_kernel<<<(int)blocks, 256, 0, st>>>(nrows, nnz_len, rowptr, tile_nnz, ntiles, tile_row,
                                                 plan_flags, status);
    return (int)cudaGetLastError();
}

int launch_csr_spmv(cudaStream_t st, int assoc, int nrows, int ncols, int nnz_len,
                    const int* rowptr, const int* col, const float* val, const float* x, float* y,
                    const int* tile_row, int ntiles, const unsigned* plan_flags, unsigned* status) {
    if (nrows <= 0) return 0;
    int grid = ntiles;
    if (assoc)
        csr_stream_kernel<true><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val,
                                                            x, y, tile_row, ntiles, plan_flags, status);
    else
        csr_stream_kernel<false><<<grid, SPMV_THREADS, 0, st>>>(nrows, ncols, nnz_len, rowptr, col, val,
                                                             x, y, tile_row, ntiles, plan_flags, status);
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

int csr_tile_nnz() { return SPMV_CHUNK; }
