/* ORACLE / TEST INFRASTRUCTURE ONLY — see pencil_oracle.h.
 *
 * Each function restates, for one PENCIL fixture, what pencil::Interpreter::call
 * (interp.cpp:95-99) computes when it walks that fixture's AST:
 *   - `for` bounds are evaluated once, then the body runs lo..hi-1 in order
 *     (interp.cpp:207-217);
 *   - float-typed scalars start as fp64 0.0 and every float operation is an fp64
 *     operation on the stored values (Decl interp.cpp:152-166, arith interp.cpp:33-48);
 *     an fp32 array element is loaded as the exact double of its fp32 value;
 *   - int arithmetic is int64 with C truncating `/` and a division-by-zero fault
 *     (interp.cpp:49-64);
 *   - `s += e` is s = s + e (apply_compound, interp.cpp:74-83);
 *   - every array load/store is bounds-checked against the stored array's length and
 *     faults with E-INTERP (interp.cpp:186-195, 267-282).
 * The outer (independent) loops are split across OpenMP threads purely for speed:
 * each output element is still produced by one thread in the interpreter's order,
 * so the result does not depend on the thread count.  Compiled with
 * -ffp-contract=off so no product/sum pair is fused (the interpreter rounds both).
 */
#include "pencil_oracle.h"

#include <stddef.h>

/* gemv.pencil.c: y[i] = alpha * s + beta * y[i], s = sum_j A[i*n+j]*x[j] */
int oracle_gemv(int m, int n, double alpha, double beta, const float* A, const float* x,
                const float* y_in, double* y_out) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < m; i++) {
        double s = 0.0;                                   /* float s; s = 0.0; */
        for (long long j = 0; j < n; j++)
            s = s + (double)A[i * n + j] * (double)x[j];  /* s += A[i*n+j] * x[j] */
        y_out[i] = alpha * s + beta * (double)y_in[i];
    }
    return 0;
}

/* gemv_t.pencil.c: y[j*incy] = alpha * sum_i A[i*lda+j]*x[i*incx] + beta * y[j*incy] */
int oracle_gemv_t(int m, int n, int lda, int incx, int incy, double alpha, double beta,
                  const float* A, long long a_len, const float* x, long long x_len,
                  const float* y_in, long long y_len, double* y_out) {
    int fault = 0;
    for (long long t = 0; t < y_len; t++) y_out[t] = (double)y_in[t];
#pragma omp parallel for schedule(static) reduction(| : fault)
    for (long long j = 0; j < n; j++) {
        double s = 0.0;
        int bad = 0;
        for (long long i = 0; i < m && !bad; i++) {
            long long ia = i * lda + j, ix = i * incx;
            if (ia < 0 || ia >= a_len || ix < 0 || ix >= x_len) { bad = 1; break; }
            s = s + (double)A[ia] * (double)x[ix];
        }
        long long iy = j * incy;
        if (bad || iy < 0 || iy >= y_len) { fault |= 1; continue; }
        y_out[iy] = alpha * s + beta * (double)y_in[iy];
    }
    return fault;
}

/* dot.pencil.c: s += x[i]*y[i]; return s (the fp64 value, not narrowed: interp.cpp:235-238) */
int oracle_dot(int n, const float* x, const float* y, double* out) {
    double s = 0.0;
    for (long long i = 0; i < n; i++) s = s + (double)x[i] * (double)y[i];
    *out = s;
    return 0;
}

/* axpy.pencil.c: y[i] = a * x[i] + y[i] */
int oracle_axpy(int n, double a, const float* x, const float* y_in, double* y_out) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; i++) y_out[i] = a * (double)x[i] + (double)y_in[i];
    return 0;
}

/* spmv.pencil.c (spmv_vec / spmv_inline / spmv+spmv_row): the three spellings execute
 * identically in the interpreter: for k in [rowptr[i], rowptr[i+1]): s += val[k]*x[col[k]] */
int oracle_spmv(int nrows, int ncols, int nnz, const int* rowptr, const int* col,
                const float* val, const float* x, double* y_out) {
    int fault = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : fault)
    for (long long i = 0; i < nrows; i++) {
        long long lo = rowptr[i], hi = rowptr[i + 1];
        double s = 0.0;
        for (long long k = lo; k < hi; k++) {
            if (k < 0 || k >= nnz) { fault |= 1; break; }
            long long c = col[k];
            if (c < 0 || c >= ncols) { fault |= 1; break; }
            s = s + (double)val[k] * (double)x[c];
        }
        y_out[i] = s;
    }
    return fault;
}

/* conv5x5.pencil.c conv5x5_u8: clamp-to-edge, int64 accumulate, (acc + scale/2)/scale
 * truncating toward zero, saturate to [0, 255]. */
int oracle_conv5x5_u8(int h, int w, int scale, const int* img, const int* k, long long* out) {
    if (scale == 0 && h > 0 && w > 0) return 1; /* "division by zero" (interp.cpp:56-57) */
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < h; i++) {
        for (long long j = 0; j < w; j++) {
            long long acc = 0;
            for (int di = 0; di < 5; di++)
                for (int dj = 0; dj < 5; dj++) {
                    long long r = i + di - 2, c = j + dj - 2;
                    if (r < 0) r = 0;
                    if (r > h - 1) r = h - 1;
                    if (c < 0) c = 0;
                    if (c > w - 1) c = w - 1;
                    acc = acc + (long long)k[di * 5 + dj] * (long long)img[r * w + c];
                }
            acc = (acc + scale / 2) / scale;
            if (acc < 0) acc = 0;
            if (acc > 255) acc = 255;
            out[i * w + j] = acc;
        }
    }
    return 0;
}

/* conv5x5.pencil.c conv5x5_f32: interior pixels only; the border of out is not stored to. */
int oracle_conv5x5_f32(int h, int w, const float* img, const float* k, const float* out_in,
                       double* out) {
    for (long long t = 0; t < (long long)h * w; t++) out[t] = (double)out_in[t];
#pragma omp parallel for schedule(static)
    for (long long i = 2; i < h - 2; i++) {
        for (long long j = 2; j < w - 2; j++) {
            double acc = 0.0;
            for (int di = 0; di < 5; di++)
                for (int dj = 0; dj < 5; dj++)
                    acc = acc + (double)k[di * 5 + dj] * (double)img[(i + di - 2) * w + (j + dj - 2)];
            out[i * w + j] = acc;
        }
    }
    return 0;
}

/* gemm.pencil.c: C[i*n+j] = alpha * sum_p A[i*k+p]*B[p*n+j] + beta * C[i*n+j] */
int oracle_gemm(int m, int n, int k, double alpha, double beta, const float* A, const float* B,
                const float* C_in, double* C_out) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < m; i++) {
        for (long long j = 0; j < n; j++) {
            double s = 0.0;
            for (long long p = 0; p < k; p++) s = s + (double)A[i * k + p] * (double)B[p * n + j];
            C_out[i * n + j] = alpha * s + beta * (double)C_in[i * n + j];
        }
    }
    return 0;
}

/* ---- fp32 semantics of the reference-EMITTED C (emit_openmp output compiled as written,
 * -ffp-contract=off, oracle/Makefile OMP_FLAGS): every float `*` and `+` rounds to fp32 on
 * its own (C99 with FLT_EVAL_METHOD 0), sums in source order.  Used to pin the emitted
 * library, and as the bit-exact target of the source-order CUDA schedules. */
int oracle_spmv_f32(int nrows, int ncols, int nnz, const int* rowptr, const int* col,
                    const float* val, const float* x, float* y_out) {
    int fault = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : fault)
    for (long long i = 0; i < nrows; i++) {
        float s = 0.0f;
        for (long long k = rowptr[i]; k < rowptr[i + 1]; k++) {
            if (k < 0 || k >= nnz || col[k] < 0 || col[k] >= ncols) { fault |= 1; break; }
            float p = val[k] * x[col[k]];
            s = s + p;
        }
        y_out[i] = s;
    }
    return fault;
}

int oracle_conv5x5_f32_f32(int h, int w, const float* img, const float* k, float* out) {
#pragma omp parallel for schedule(static)
    for (long long i = 2; i < h - 2; i++)
        for (long long j = 2; j < w - 2; j++) {
            float acc = 0.0f;
            for (int di = 0; di < 5; di++)
                for (int dj = 0; dj < 5; dj++) {
                    float p = k[di * 5 + dj] * img[(i + di - 2) * w + (j + dj - 2)];
                    acc = acc + p;
                }
            out[i * w + j] = acc;
        }
    return 0;
}

int oracle_axpy_f32(int n, float a, const float* x, float* y) {
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < n; i++) {
        float p = a * x[i];
        y[i] = p + y[i];
    }
    return 0;
}
