// Internal launcher interface between the C++ host runtime (runtime.cpp) and the CUDA
// translation units.  All launchers are stream-ordered and never synchronize; they return
// a cudaError_t value (0 = launched).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

// k_blas.cu
int launch_gemv(cudaStream_t st, int m, int n, float alpha, float beta, const float* A,
                const float* x, float* y);
int launch_gemv_t(cudaStream_t st, int m, int n, int lda, int incx, int incy, float alpha,
                  float beta, const float* A, const float* x, float* y, float* partial,
                  unsigned* counters);
size_t gemv_t_partial_elems(int m, int n);
size_t gemv_t_counter_elems(int n);
int launch_dot(cudaStream_t st, long long n, const float* x, const float* y, float* result,
               double* partial, unsigned* counter);
size_t dot_partial_elems();
int launch_axpy(cudaStream_t st, long long n, float a, const float* a_dev, const float* x,
                float* y);

// k_spmv.cu
// rs_bits (optional, csr_rs_words(nnz) words): the row-start bitmap of the segmented executor
// The plan's tiles: windows of tile_nnz non-zeros up to tail_start, then of tail_nnz (a tapered
// tail, so that the warps drawing the last tickets finish together); ntiles in all.
struct TileSchedule {
    int tile_nnz = 1;
    long long tail_start = 0;
    int tail_nnz = 1;
    int ntiles = 1;
};
TileSchedule csr_tile_schedule(int mode, int nnz_len);
int launch_csr_plan(cudaStream_t st, int nrows, int nnz_len, const int* rowptr, const TileSchedule& ts,
                    int* tile_row, unsigned* plan_flags, unsigned* rs_bits, unsigned* status);
size_t csr_rs_words(int nnz_len);
// plans with empty rows: ord (nrows + 1 ints) / rowmap (one int per non-empty row), bsum scratch
int launch_csr_ordinals(cudaStream_t st, int nrows, const int* rowptr, int* ord, int* rowmap, int* bsum);
size_t csr_ord_scratch_ints();
// The segmented executor's plan data: rs_bits = the row-start bitmap when it may run (monotone
// rowptr, aligned col / val), else NULL; for plans with empty rows, ord / rowmap (else NULL) — the
// executor then writes only the non-empty rows: the caller zeroes y first.
struct SegPlan {
    const unsigned* rs_bits = nullptr;
    const int* ord = nullptr;
    const int* rowmap = nullptr;
};
// tk: the per-(device, stream) tile-ticket word (zero between launches; the kernels re-arm it)
int launch_csr_spmv(cudaStream_t st, int assoc, int nrows, int ncols, int nnz_len,
                    const int* rowptr, const int* col, const float* val, const float* x, float* y,
                    const int* tile_row, int ntiles, const unsigned* plan_flags, const SegPlan& seg,
                    unsigned* tk, unsigned* status);
int launch_csr_generic(cudaStream_t st, int nrows, int ncols, int nnz_len, const int* rowptr,
                       const int* col, const float* val, const float* x, float* y,
                       unsigned* status);
// fused SpMV -> all-gather of y: every row result is also stored to `n` peer buffers (NVLink
// peer mappings, each already offset to this rank's slot) or, when mc is set, once to an NVLS
// multicast address that replicates it to every rank
#define PENCIL_MAX_PEERS 8
struct PeerSet {
    float* p[PENCIL_MAX_PEERS];
    float* mc;
    int n;
};
int launch_csr_spmv_dist(cudaStream_t st, int assoc, int nrows, int ncols, int nnz_len,
                         const int* rowptr, const int* col, const float* val, const float* x, float* y,
                         const int* tile_row, int ntiles, const unsigned* plan_flags, const SegPlan& seg,
                         unsigned* tk, unsigned* status, const PeerSet& peers);

// k_conv.cu  (taps are host arrays, passed to the kernels by value)
int launch_conv5x5_f32(cudaStream_t st, int h, int w, const float* img, const float* k25,
                       float* out);
int launch_conv5x5_u8(cudaStream_t st, int h, int w, int scale, const int* img, const int* k25,
                      int* out);
int launch_conv5x5_u8_bytes(cudaStream_t st, int h, int w, int scale, const unsigned char* img,
                            const int* k25, unsigned char* out);
// output rows [lo, hi) of the h-row image, when a SWAR kernel applies (cudaErrorNotSupported otherwise)
int launch_conv5x5_u8_bytes_rows(cudaStream_t st, int h, int w, int scale, const unsigned char* img, const int* k25,
                                 unsigned char* out, int lo, int hi);
bool conv5x5_u8_bytes_rows_ok(int h, int w, int scale, const int* k25);
// band-sharded sweeps (k_stencil.cu): rows -2, -1 / h, h + 1 of the band through top / bot
int launch_conv5x5_u8_band(cudaStream_t st, int h, int w, int scale, const int* img, const int* const* top,
                           const int* const* bot, const int* k25, int* out);
int launch_conv5x5_f32_band(cudaStream_t st, int h, int w, int out_lo, int out_hi, const float* img,
                            const float* const* top, const float* const* bot, const float* k25, float* out);

// k_gemm.cu
int launch_gemm(cudaStream_t st, int m, int n, int k, float alpha, float beta, const float* A, long long lda,
                const float* B, long long ldb, float* C, long long ldc, void* workspace, size_t workspace_bytes);
size_t gemm_workspace_bytes(int m, int n, int k, const float* A, long long lda, const float* B, long long ldb);

// k_micro.cu (measurement probes, not PENCIL kernels)
int launch_micro_gather(cudaStream_t st, int mode, long long n, const int* idx, const float* table,
                        float* out);
int launch_micro_copy(cudaStream_t st, long long n, const float* src, float* dst);
int launch_micro_gather_val(cudaStream_t st, long long n, const int* idx, const float* val, const float* table,
                            float* out);
int launch_micro_l2_flush(cudaStream_t st, long long n, float* buf);
