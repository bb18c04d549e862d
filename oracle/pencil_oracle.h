/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * C restatement of the reference interpreter's semantics for the PENCIL kernel
 * fixtures (paper_1302_5586_b200/pencil/*.pencil.c).  pencil::Interpreter
 * (/root/reference/proj/core/src/interp.cpp) holds every value as int64 or fp64
 * (interp.hpp:12, arith at interp.cpp:27-72), so these functions take the fp32/int32
 * inputs the CUDA path sees and return fp64/int64 outputs computed in the
 * interpreter's evaluation order.  Pinned bit-for-bit against the real interpreter
 * (oracle/_ref/ref_driver run) by tests/test_oracle.py on tests/golden/*.npz.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this; the product library never does.
 *
 * Every function returns 0, or 1 where the interpreter would throw
 * PencilError("E-INTERP", ...) (out-of-bounds load, division by zero).
 */
#ifndef PENCIL_ORACLE_H
#define PENCIL_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

int oracle_gemv(int m, int n, double alpha, double beta, const float* A, const float* x,
                const float* y_in, double* y_out);
int oracle_gemv_t(int m, int n, int lda, int incx, int incy, double alpha, double beta,
                  const float* A, long long a_len, const float* x, long long x_len,
                  const float* y_in, long long y_len, double* y_out);
int oracle_dot(int n, const float* x, const float* y, double* out);
int oracle_axpy(int n, double a, const float* x, const float* y_in, double* y_out);
int oracle_spmv(int nrows, int ncols, int nnz, const int* rowptr, const int* col,
                const float* val, const float* x, double* y_out);
int oracle_conv5x5_u8(int h, int w, int scale, const int* img, const int* k, long long* out);
int oracle_conv5x5_f32(int h, int w, const float* img, const float* k, const float* out_in,
                       double* out);
int oracle_gemm(int m, int n, int k, double alpha, double beta, const float* A, const float* B,
                const float* C_in, double* C_out);

/* fp32 semantics of the reference-emitted C, compiled as written (see pencil_oracle.c) */
int oracle_spmv_f32(int nrows, int ncols, int nnz, const int* rowptr, const int* col,
                    const float* val, const float* x, float* y_out);
int oracle_conv5x5_f32_f32(int h, int w, const float* img, const float* k, float* out);
int oracle_axpy_f32(int n, float a, const float* x, float* y);

#ifdef __cplusplus
}
#endif
#endif
