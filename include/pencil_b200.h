/* pencil_b200.h — C ABI of the B200-native execution backend for PENCIL kernels.
 *
 * Reference boundary (arxiv/paper_1302_5586 reference under /root/reference, read-only):
 * the reference's CPU-parallel code generator emit_openmp (proj/core/src/pretty.cpp:472-531)
 * prints every PENCIL array parameter `T a[restrict const static e]` (Printer::param,
 * pretty.cpp:221-233); C decays it to `T *a`, scalars stay int/float, returns stay
 * void/int/float.  Section 1 exports exactly those signatures for the kernel fixtures in
 * paper_1302_5586_b200/pencil/*.pencil.c, so a program that linked the emitted-OpenMP object
 * links this library instead.  Nothing here throws across the ABI.
 */
#ifndef PENCIL_B200_H
#define PENCIL_B200_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ===== 1. Drop-in entry points (replace the emitted-OpenMP functions) ==================
 * Pointers may be host memory (pageable or pinned; copied in/out around the call, the call
 * returns when results are back in host memory) or CUDA device memory on the current
 * device (used in place, no copies; the call still returns when the work is complete).
 * `restrict` (PENCIL rule R1, compliance.cpp:152-164) guarantees the arrays do not alias.
 * On failure the outputs are unspecified and pencil_cuda_last_status() != 0. */

/* gemv.pencil.c    <- replaces emitted `void gemv(int, int, float, float, float *, float *, float *)` */
void gemv(int m, int n, float alpha, float beta, float* A, float* x, float* y);
/* gemv_t.pencil.c  (VOBLA transposed / strided view) */
void gemv_t(int m, int n, int lda, int incx, int incy, float alpha, float beta, float* A,
            float* x, float* y);
/* dot.pencil.c */
float dot(int n, float* x, float* y);
/* axpy.pencil.c */
void axpy(int n, float a, float* x, float* y);
/* spmv.pencil.c: spmv_vec (row reduction licensed), spmv_inline (row sum in source order),
 * spmv (row loop over the ACCESS-summarised spmv_row) — identical signatures */
void spmv_vec(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y);
void spmv_inline(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y);
void spmv(int nrows, int ncols, int nnz, int* rowptr, int* col, float* val, float* x, float* y);
void spmv_row(int nrows, int ncols, int nnz, int i, int* rowptr, int* col, float* val, float* x, float* y);
/* conv5x5.pencil.c (u8 image semantics held in int, clamp-to-edge; fp32 interior-only) */
void conv5x5_u8(int h, int w, int scale, int* img, int* k, int* out);
void conv5x5_f32(int h, int w, float* img, float* k, float* out);
/* gemm.pencil.c (fp32 via 3xTF32 on tcgen05 tensor cores) */
void gemm(int m, int n, int k, float alpha, float beta, float* A, float* B, float* C);

/* ===== 2. Status channel (mirrors PencilError codes, diag.hpp:44-55) ===================== */
enum pencil_status {
    PENCIL_OK = 0,
    PENCIL_E_INTERP = 1,      /* runtime fault: out-of-bounds load, division by zero, bad call */
    PENCIL_E_ARG = 2,         /* invalid argument (negative extent, null pointer, wrong dtype) */
    PENCIL_E_CUDA = 3,        /* CUDA runtime error */
    PENCIL_E_NOMEM = 4,       /* device allocation failed */
    PENCIL_E_UNSUPPORTED = 5, /* no schedule for this nest / shape */
    /* OP2 mesh-model codes (op2.hpp:79-81, op2.cpp:14-17, 205, 226, 233) */
    PENCIL_E_OP2_SHAPE = 6,   /* malformed document, wrong table/data lengths, unknown names */
    PENCIL_E_OP2_RANGE = 7,   /* map entry or arg offset out of range */
    PENCIL_E_OP2_KERNEL = 8,  /* kernel missing, unparsable, or signature != 2m+n */
    PENCIL_E_OP2_CONFLICT = 9, /* a dat both incremented and written in one par_loop */
    /* OptiML construct codes (optiml.hpp:27-29) */
    PENCIL_E_OPTIML_SHAPE = 10, /* malformed construct, unknown kind or variant */
    PENCIL_E_OPTIML_RANGE = 11  /* empty sum range */
};
int pencil_cuda_last_status(void);
const char* pencil_cuda_last_error(void); /* "E-INTERP: load from x[...] is out of bounds" style */
void pencil_cuda_clear_status(void);
const char* pencil_status_code(int status); /* "E-INTERP", "E-ARG", ... */

/* ===== 3. Device-resident, stream-ordered API (no host synchronization) ==================
 * `stream` is a cudaStream_t of the current device (0 = the legacy default stream).
 * Device faults (E-INTERP analogues) accumulate in a per-(device, stream) status word read and
 * cleared by pencil_sync_status(stream). Every device word a launch mutates (fault word, SpMV
 * tile tickets, gemv_t last-CTA counters) is per (device, stream), so calls on different streams
 * — one CSR plan included — run concurrently without sharing state.
 * Return value: pencil_status of the launch itself. */
typedef void* pencil_stream_t;
int pencil_gemv_dev(pencil_stream_t s, int m, int n, float alpha, float beta, const float* A,
                    const float* x, float* y);
int pencil_gemv_t_dev(pencil_stream_t s, int m, int n, int lda, int incx, int incy, float alpha,
                      float beta, const float* A, const float* x, float* y);
int pencil_dot_dev(pencil_stream_t s, long long n, const float* x, const float* y, float* result_dev);
int pencil_axpy_dev(pencil_stream_t s, long long n, float a, const float* x, float* y);
/* axpy with the scalar read from device memory (e.g. the result of pencil_dot_dev) */
int pencil_axpy_dev_ptr(pencil_stream_t s, long long n, const float* a_dev, const float* x, float* y);
int pencil_conv5x5_u8_dev(pencil_stream_t s, int h, int w, int scale, const int* img,
                          const int* k_host, int* out);
/* packed 8-bit image variant (1 byte per pixel, same arithmetic as conv5x5_u8) */
int pencil_conv5x5_u8_bytes_dev(pencil_stream_t s, int h, int w, int scale, const uint8_t* img,
                                const int* k_host, uint8_t* out);
/* the packed 8-bit stencil on host arrays (copied in / out like the §1 calls; pageable arrays of
 * 4 MB and more through the library's staging ring) or device arrays (used in place) */
int pencil_conv5x5_u8_bytes(int h, int w, int scale, const uint8_t* img, const int* k, uint8_t* out);
int pencil_conv5x5_f32_dev(pencil_stream_t s, int h, int w, const float* img, const float* k_host,
                           float* out);
/* Band-sharded 5x5 stencils (multi-GPU row bands; the halo exchange is fused into the sweep):
 * the band's own h rows at img / out; top[0], top[1] = rows -2, -1 and bot[0], bot[1] = rows h,
 * h + 1 as device pointers — the neighbour ranks' edge rows through their peer mappings (NVLink),
 * or the band's own first / last row repeated at the image's top / bottom (clamp-to-edge).  The
 * f32 form writes band rows [out_lo, out_hi) (the image interior).  Needs w % 4 == 0 and 16-byte
 * aligned rows (else PENCIL_E_ARG).  Results are the rows of the whole-image call, bit for bit.
 * Replaces the exchange + compute pair of the row-band path (conv5x5 row). */
int pencil_conv5x5_u8_band_dev(pencil_stream_t s, int h, int w, int scale, const int* img,
                               const int* const* top, const int* const* bot, const int* k_host, int* out);
int pencil_conv5x5_f32_band_dev(pencil_stream_t s, int h, int w, int out_lo, int out_hi, const float* img,
                                const float* const* top, const float* const* bot, const float* k_host,
                                float* out);
int pencil_gemm_dev(pencil_stream_t s, int m, int n, int k, float alpha, float beta, const float* A,
                    const float* B, float* C);
/* gemm on strided views: A m x k with row pitch lda, B k x n pitch ldb, C m x n pitch ldc (a tile of a
 * larger C, a column panel of B — the views of the distribution plan's gemm split, §10); the
 * operands are read in place by TMA when base and pitch are 16-byte multiples */
int pencil_gemm_strided_dev(pencil_stream_t s, int m, int n, int k, float alpha, float beta, const float* A,
                            long long lda, const float* B, long long ldb, float* C, long long ldc);

/* CSR inspector/executor: the plan is built once per sparsity structure (one pass over rowptr)
 * and reused by every SpMV on that structure.  mode: 0 = row sums in source order (spmv_inline,
 * spmv), 1 = reassociation licensed (spmv_vec). */
typedef struct pencil_csr_plan* pencil_csr_plan_t;
int pencil_csr_plan_create(pencil_stream_t s, int nrows, int ncols, int nnz, const int* rowptr_dev,
                           int mode, pencil_csr_plan_t* out);
int pencil_csr_plan_destroy(pencil_csr_plan_t plan);
int pencil_csr_plan_info(pencil_csr_plan_t plan, int* ntiles, int* tile_nnz);
int pencil_spmv_dev(pencil_stream_t s, pencil_csr_plan_t plan, const int* rowptr, const int* col,
                    const float* val, const float* x, float* y);

/* Fused SpMV -> all-gather of y (one step of a row-sharded iterative SpMV): as
 * pencil_spmv_dev, and every row result y[i] is also stored to peers[q][i] for q < npeers
 * (device-visible pointers — NVLink peer mappings of the other ranks' gathered-vector buffers,
 * each offset to this rank's slot) or, when mc is not NULL, once to the NVLS multicast address
 * mc + i, which the switch replicates to every rank.  The stores are fenced at system scope
 * before the launch retires; the caller orders the consumers after it with a cross-rank
 * barrier on `s`.  npeers <= 8. */
int pencil_spmv_dev_dist(pencil_stream_t s, pencil_csr_plan_t plan, const int* rowptr, const int* col,
                         const float* val, const float* x, float* y, float* const* peers, int npeers,
                         float* mc);

/* synchronize `s`, return and clear the device fault word (PENCIL_OK or PENCIL_E_INTERP) */
int pencil_sync_status(pencil_stream_t s);

/* ===== 4. Name-dispatch launch layer — mirror of pencil::Interpreter (interp.hpp:27-72) ===== */
enum pencil_dtype { PENCIL_INT32 = 0, PENCIL_FLOAT32 = 1, PENCIL_FLOAT64 = 2, PENCIL_UINT8 = 3 };
enum pencil_arg_kind { PENCIL_ARG_INT = 0, PENCIL_ARG_FLOAT = 1, PENCIL_ARG_ARRAY = 2 };
typedef struct {
    int kind;            /* pencil_arg_kind */
    long long i;         /* PENCIL_ARG_INT */
    double f;            /* PENCIL_ARG_FLOAT */
    const char* array;   /* PENCIL_ARG_ARRAY: store name (Interpreter::Arg::array) */
} pencil_arg;
typedef struct {
    int kind;            /* PENCIL_ARG_INT / PENCIL_ARG_FLOAT; -1 for void */
    long long i;
    double f;
} pencil_value;
typedef struct pencil_runtime* pencil_runtime_t;
pencil_runtime_t pencil_runtime_create(int device);
void pencil_runtime_destroy(pencil_runtime_t rt);
/* Interpreter::set_array: copy host data into a named device array (replaces any previous) */
int pencil_runtime_set_array(pencil_runtime_t rt, const char* name, int dtype, const void* host,
                             long long n);
/* bind existing device memory under a name (no copy; caller keeps ownership) */
int pencil_runtime_bind_array(pencil_runtime_t rt, const char* name, int dtype, void* dev,
                              long long n);
/* Interpreter::arrays()[name]: copy back to host (n elements) */
int pencil_runtime_get_array(pencil_runtime_t rt, const char* name, void* host, long long n);
int pencil_runtime_array_info(pencil_runtime_t rt, const char* name, int* dtype, long long* n,
                              void** dev);
/* Interpreter::call: name -> kernel through the mapper's schedule; synchronous */
int pencil_runtime_call(pencil_runtime_t rt, const char* fn, int nargs, const pencil_arg* args,
                        pencil_value* ret);
/* the fp-reduction-reorders-results flag of the last call (pencilc.cpp:157-161 analogue) */
int pencil_runtime_fp_reordered(pencil_runtime_t rt);
/* the kernel variant the mapper chose for the last call (pencil_schedule.kernel): the call
 * launches that kernel — the CSR fixtures, e.g., fold their rows in source order or
 * reassociated according to the inner loop's role, not according to the function name */
const char* pencil_runtime_last_kernel(pencil_runtime_t rt);

/* ===== 5. Mapper: loop verdicts -> grid/block/tile schedule ==============================
 * Verdicts are the reference analyzer's (depanalysis.hpp:14 Verdict, same numbering). */
enum pencil_verdict {
    PENCIL_PARALLEL = 0,
    PENCIL_PARALLEL_WITH_REDUCTION = 1,
    PENCIL_SERIAL = 2,
    PENCIL_UNKNOWN = 3,
    PENCIL_ASSUMED_PARALLEL = 4
};
typedef struct {
    int loop_id;
    int depth;           /* nesting depth within its function (0 = outermost) */
    int verdict;         /* pencil_verdict */
    char reduction_op;   /* '+', '*', 'M' (max), 'm' (min) or 0 */
} pencil_loop_verdict;
enum pencil_dim_role { PENCIL_DIM_GRID = 0, PENCIL_DIM_TILE = 1, PENCIL_DIM_REDUCE = 2, PENCIL_DIM_SEQ = 3 };
typedef struct {
    int nloops;
    int role[8];         /* pencil_dim_role per depth */
    int grid_dims;       /* loops mapped to the launch grid */
    int reassociates;    /* a reduction is split across threads (fp rounding may change) */
    char kernel[48];     /* chosen kernel variant */
} pencil_schedule;
/* map the verdicts of one PENCIL function's loop nest (depth-ordered) */
int pencil_map_nest(const char* fn, const pencil_loop_verdict* loops, int nloops, pencil_schedule* out);
/* the verdict table compiled into the library for a fixture function (from the reference
 * analyzer); returns the number of loops written (<= cap), or -1 if unknown */
int pencil_fixture_verdicts(const char* fn, pencil_loop_verdict* out, int cap);

/* ===== 6. Multi-GPU partitioning (host-only; used by one-process-per-GPU drivers) ========= */
/* row blocks of a CSR matrix balanced by non-zeros: bounds[0..nshards], bounds[0]=0, bounds[nshards]=nrows */
int pencil_shard_rows_by_nnz(const int* rowptr, int nrows, int nshards, int* bounds);
/* equal row bands of h rows (stencils); halo rows needed above/below each band */
int pencil_shard_bands(int h, int nshards, int* bounds);
/* 2-D tile grid for gemm across nshards GPUs: grid_rows * grid_cols == nshards, tiles as square as possible */
int pencil_shard_gemm_grid(int m, int n, int nshards, int* grid_rows, int* grid_cols);

/* ===== 7. Introspection / measurement =================================================== */
const char* pencil_version(void);
/* bytes the last drop-in call on this thread moved host->device and device->host */
int pencil_last_transfer_bytes(long long* h2d, long long* d2h);
int pencil_l2_flush(pencil_stream_t s); /* write a buffer larger than L2 (timing hygiene) */
int pencil_micro_gather(pencil_stream_t s, int mode, long long n, const int* idx,
                        const float* table, float* out);
int pencil_micro_copy(pencil_stream_t s, long long n, const float* src, float* dst);
/* SpMV data path without rows: stream idx + val, gather table[idx] (roofline probe) */
int pencil_micro_gather_val(pencil_stream_t s, long long n, const int* idx, const float* val,
                            const float* table, float* out);

/* ===== 8. OP2 mesh loops on the GPU ======================================
 * The reference's mesh model (core/include/pencil/op2.hpp; JSON format of docs/op2-input.md)
 * executed on the device with the sequential semantics of interpret_op2_reference
 * (core/src/op2.cpp:388-429).  Kernels are compiled from their PENCIL source (NVRTC, sm_100a);
 * dats stay device-resident between runs. */
typedef struct pencil_op2_model* pencil_op2_t;
/* load_op2_model (op2.hpp:79) + kernel parse/signature/conflict checks of lower_op2_model;
 * NULL on error (status E-OP2-SHAPE / -RANGE / -KERNEL / -CONFLICT / E-UNSUPPORTED) */
pencil_op2_t pencil_op2_load(const char* json_text);
void pencil_op2_free(pencil_op2_t m);
int pencil_op2_num_loops(pencil_op2_t m);
/* schedule of par_loop `loop`: 0 parallel (OP_INC as atomic adds), 1 iteration levels,
 * 2 serial; levels = launches for strategy 1 (known after pencil_op2_prepare) */
int pencil_op2_loop_info(pencil_op2_t m, int loop, int* strategy, int* levels);
int pencil_op2_prepare(pencil_op2_t m);        /* compile + upload (also done by the first run) */
int pencil_op2_run(pencil_op2_t m);            /* every par_loop in order; synchronous, faults -> E-INTERP */
int pencil_op2_run_loop_async(pencil_op2_t m, int loop); /* enqueue one par_loop on the model's stream */
int pencil_op2_sync(pencil_op2_t m);           /* wait for the model's stream, report faults */
long long pencil_op2_dat_size(pencil_op2_t m, const char* dat); /* values (set size x dim), -1 if unknown */
int pencil_op2_get_dat(pencil_op2_t m, const char* dat, long long* out, long long n);
int pencil_op2_set_dat(pencil_op2_t m, const char* dat, const long long* in, long long n);
const char* pencil_op2_cuda_source(pencil_op2_t m); /* generated CUDA (inspection) */
const char* pencil_op2_lowered(pencil_op2_t m);     /* the model lowered to PENCIL drivers (append_driver) */
void* pencil_op2_stream(pencil_op2_t m);            /* cudaStream_t the model runs on */

/* ===== 9. PENCIL units on the GPU: the general mapper (emit_cuda) ============
 * Any compliant unit, compiled for sm_100a (NVRTC) with the reference Interpreter's value
 * semantics; top-level loops of the called function with `#pragma pencil independent` run one
 * iteration per thread, `#pragma pencil reduction (op: v)` loops add a fixed-order combine, other
 * statements run in order on one device thread (jit.cpp). Surface of pencil::Interpreter. */
typedef struct pencil_jit* pencil_jit_t;
pencil_jit_t pencil_jit_load(const char* source);  /* NULL on error (E-ARG "E-SYNTAX: ...", E-UNSUPPORTED) */
void pencil_jit_free(pencil_jit_t j);
int pencil_jit_set_array(pencil_jit_t j, const char* name, int dtype, const void* host, long long n);
long long pencil_jit_array_size(pencil_jit_t j, const char* name);
/* values as fp64 + per-element is_double flag (+ exact int64 of integer elements, optional) */
int pencil_jit_get_array(pencil_jit_t j, const char* name, double* out, unsigned char* is_double,
                         long long* ints, long long n);
int pencil_jit_call(pencil_jit_t j, const char* fn, int nargs, const pencil_arg* args, pencil_value* ret);
/* per top-level segment of fn: 'S' serial, 'P' parallel loop, 'R' parallel loop with reduction */
int pencil_jit_schedule(pencil_jit_t j, const char* fn, char* out, int cap);
const char* pencil_jit_cuda_source(pencil_jit_t j);
/* access summary of fn's array parameters: "name=r|w|rw|-[!]" comma separated,
 * "!" = written in full before any read; returns the length or -1 */
int pencil_jit_access(pencil_jit_t j, const char* fn, char* out, int cap);
/* call on HOST arrays (args[i] of kind PENCIL_ARG_ARRAY use host[i], dtypes[i], counts[i]) with
 * uploads / downloads planned from the access summary; bytes moved: pencil_jit_last_traffic */
int pencil_jit_call_host(pencil_jit_t j, const char* fn, int nargs, const pencil_arg* args, void* const* host,
                         const int* dtypes, const long long* counts, pencil_value* ret);
int pencil_jit_last_traffic(pencil_jit_t j, long long* h2d, long long* d2h);
/* Interpreter::set_rand_sequence: rand() returns these first, then the interpreter's LCG */
int pencil_jit_set_rand_sequence(pencil_jit_t j, const long long* values, long long n);
/* Interpreter::set_array with the interpreter's Value per element (int64 or fp64): element i is
 * dbls[i] when is_double[i], else ints[i] (arrays may mix both, as the interpreter's do) */
int pencil_jit_set_array_values(pencil_jit_t j, const char* name, const long long* ints, const double* dbls,
                                const unsigned char* is_double, long long n);
/* Interpreter::enable_trace / trace (interp.hpp:45-46, MemTrace interp.hpp:17-21): with the trace
 * on, calls run every statement on one device thread in the interpreter's order and record each
 * in-bounds load / store of a named store array (store name, flat index, is_write) — local arrays
 * and *p dereferences are not recorded, as in the interpreter.  Records accumulate across calls. */
int pencil_jit_enable_trace(pencil_jit_t j, int on);
long long pencil_jit_trace_size(pencil_jit_t j);
/* records [first, first + n): arrays[r] points at the store name (valid while j lives) */
int pencil_jit_trace_get(pencil_jit_t j, long long first, long long n, const char** arrays, long long* index,
                         unsigned char* is_write);
int pencil_jit_trace_clear(pencil_jit_t j);
/* OptiML construct (docs/op2-input.md; load_optiml_construct + lower_optiml, optiml.hpp:27-41)
 * lowered to a PENCIL unit for pencil_jit_load: returns the text length (cap 0 sizes the buffer)
 * or -1 (E-OPTIML-SHAPE / E-OPTIML-RANGE) */
long long pencil_optiml_lower(const char* json_text, char* out, long long cap);

/* ===== 10. Array and view descriptors ===========================
 * A view is how a PENCIL nest addresses an array: element (i, j) of the view is
 * base[offset + i * stride[0] + j * stride[1]] (rank 2) or base[offset + i * stride[0]] (rank 1).
 * Views come from the symbolic affine forms of a nest's accesses (the reference's affine_form,
 * depanalysis.cpp:163-193, keeps constant coefficients only; these keep scalar parameters such
 * as lda / incx / incy and evaluate them under a call's bindings). */
typedef struct {
    void* base;            /* device pointer of the array's element 0 */
    long long offset;      /* first element of the view */
    int rank;              /* 1 or 2 */
    int dtype;             /* pencil_dtype */
    long long extent[2];   /* view shape */
    long long stride[2];   /* elements between consecutive indices of each dimension */
} pencil_view;
/* one array access of a PENCIL function: its enclosing for-loops (outermost first) with their
 * bounds under the binding, and index = offset + sum_d stride[d] * loop_d when affine */
typedef struct {
    char array[32];
    int is_write;            /* a store (a compound store also yields a load record) */
    int affine;              /* 0: the index is not affine in the enclosing loop variables */
    int nloops;
    char loop[8][16];
    long long lo[8], hi[8];  /* loop bounds under the binding (hi exclusive) */
    long long stride[8];     /* index change per unit step of loop d */
    long long offset;        /* the index with every loop variable 0 */
    char form[128];          /* symbolic form, e.g. "i*lda + j" */
} pencil_access_form;
/* accesses of `fn` in a PENCIL unit under scalar bindings names[k] = values[k]; returns the
 * number of accesses (out holds the first cap) or -1 (E-ARG / E-SYNTAX) */
int pencil_affine_accesses(const char* source, const char* fn, int nbind, const char* const* names,
                           const long long* values, pencil_access_form* out, int cap);
/* the library's own copy of a fixture unit ("gemv_t", "spmv", ... = pencil/<name>.pencil.c) */
const char* pencil_fixture_source(const char* fixture);
/* distribution plan of fn's outermost parallel loop (and the `independent` loop nested in it):
 * JSON {"function", "dims": [{"var", "kind": "parallel"|"reduction", "reduce": [...],
 * "arrays": {name: {"mode": r|w|rw, "kind": block|view|via|all, "stride", "halo": [h0, h1],
 * "inner": [...], "via"}}, "owned", "halo", "replicated", "conflicts"}]} — which arrays a split of
 * the loop shards (blocks, views, CSR ranges via a row-pointer array), which need a halo, which
 * must be replicated (all-gathered), which reduction variables need an all-reduce (distplan.cpp).
 * Returns the length (cap 0 sizes the buffer) or -1 (E-SYNTAX / no such function / no loop). */
long long pencil_dist_plan(const char* source, const char* fn, char* out, long long cap);
/* the sub-view [lo, hi) of dimension dim */
int pencil_view_slice(const pencil_view* v, int dim, long long lo, long long hi, pencil_view* out);
/* gemv_t over views (VOBLA: y(j) = alpha * sum_i A(i, j) x(i) + beta * y(j)): A rank 2 with unit
 * stride along j, x / y rank 1 with positive strides; extents must agree (E-ARG), other
 * layouts E-UNSUPPORTED.  pencil_gemv_t_dev and the drop-in gemv_t build these views from the
 * fixture's affine forms (A[i*lda + j], x[i*incx], y[j*incy]) and call this. */
int pencil_gemv_t_view_dev(pencil_stream_t s, float alpha, float beta, const pencil_view* A, const pencil_view* x,
                           const pencil_view* y);
/* the views of the gemv_t fixture's A, x, y for a call's scalars (from its affine forms) */
int pencil_gemv_t_views(int m, int n, int lda, int incx, int incy, pencil_view views[3]);

/* Array descriptors: element type, extent, a shard spec (ordered element ranges partitioning
 * [0, n), one per rank / GPU; NULL bounds = one shard = the whole array), the device pointer of
 * each shard this process can reach (its own memory, or a peer's NVLink mapping) and an optional
 * host mirror.  The Interpreter mirror's named arrays (§4) and the multi-GPU shard classes keep
 * their arrays in these. */
typedef struct pencil_array* pencil_array_t;
pencil_array_t pencil_array_create(int dtype, long long n, int nshards, const long long* bounds);
void pencil_array_destroy(pencil_array_t a);
int pencil_array_attach(pencil_array_t a, int shard, int device, void* ptr);
int pencil_array_set_mirror(pencil_array_t a, void* host);
int pencil_array_info(pencil_array_t a, int* dtype, long long* n, int* nshards, void** host);
int pencil_array_shard(pencil_array_t a, int shard, long long* lo, long long* hi, int* device, void** ptr);
/* the shard holding element index (-1 if outside) */
int pencil_array_owner(pencil_array_t a, long long index);
/* copy a shard's element range host mirror -> device (to_device 1) or back, on stream s */
int pencil_array_sync(pencil_array_t a, int shard, int to_device, pencil_stream_t s);
/* rank-1 unit-stride view of a shard's piece */
int pencil_array_view(pencil_array_t a, int shard, pencil_view* out);
/* the descriptor of an Interpreter-mirror named array (§4; owned by the runtime, NULL if unknown) */
pencil_array_t pencil_runtime_array_desc(pencil_runtime_t rt, const char* name);

#ifdef __cplusplus
}
#endif
#endif
