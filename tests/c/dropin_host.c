/* A host program written against the C ABI that the reference's emit_openmp prints for the
 * PENCIL kernels (pretty.cpp:221-233: `T a[restrict const static e]` decays to `T *`).  The same
 * source is linked twice by tests/test_dropin_c.py: against the reference's emitted-OpenMP code
 * (oracle/_ref/libpencil_omp_outer.so, the CPU path it replaces) and against libpencil_b200.so
 * (the drop-in).  Inputs come from a fixed LCG; every input and output array is dumped to
 * argv[1] as records {name[16], dtype, count, bytes} for the comparison. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pencil_b200.h"

static uint64_t s_state = 42;
static uint32_t lcg(void) {
    s_state = s_state * 6364136223846793005ull + 1442695040888963407ull;
    return (uint32_t)(s_state >> 33);
}
static float f32(void) { return (float)(lcg() & 0xffffff) / 16777216.0f - 0.5f; }

static FILE* out;
static void dump(const char* name, int dtype, const void* p, long n) {
    char nm[16] = {0};
    strncpy(nm, name, 15);
    fwrite(nm, 1, 16, out);
    int32_t h[2] = {dtype, (int32_t)n};
    fwrite(h, 4, 2, out);
    fwrite(p, dtype == 2 ? 8 : 4, (size_t)n, out);
}
static float* fvec(long n) {
    float* v = malloc(sizeof(float) * (n ? n : 1));
    for (long i = 0; i < n; i++) v[i] = f32();
    return v;
}

static void check(const char* what) {
#ifdef PENCIL_DROPIN_B200
    if (pencil_cuda_last_status() != PENCIL_OK) {
        fprintf(stderr, "%s: %s\n", what, pencil_cuda_last_error());
        exit(3);
    }
#else
    (void)what;
#endif
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    out = fopen(argv[1], "wb");
    if (!out) return 2;
    /* gemv */
    int m = 300, n = 257;
    float *A = fvec((long)m * n), *x = fvec(n), *y = fvec(m);
    dump("gemv.A", 1, A, (long)m * n); dump("gemv.x", 1, x, n); dump("gemv.y0", 1, y, m);
    gemv(m, n, 1.5f, 0.5f, A, x, y);
    check("gemv");
    dump("gemv.y", 1, y, m);
    /* gemv_t (VOBLA strided view) */
    int tm = 65, tn = 77, lda = 80, incx = 2, incy = 3;
    float *tA = fvec((long)tm * lda), *tx = fvec((long)tm * incx), *ty = fvec((long)tn * incy);
    dump("gemvt.A", 1, tA, (long)tm * lda); dump("gemvt.x", 1, tx, (long)tm * incx);
    dump("gemvt.y0", 1, ty, (long)tn * incy);
    gemv_t(tm, tn, lda, incx, incy, 1.0f, 0.25f, tA, tx, ty);
    check("gemv_t");
    dump("gemvt.y", 1, ty, (long)tn * incy);
    /* dot, axpy */
    int nv = 100003;
    float *dx = fvec(nv), *dy = fvec(nv);
    dump("dot.x", 1, dx, nv); dump("dot.y", 1, dy, nv);
    float d = dot(nv, dx, dy);
    check("dot");
    dump("dot.r", 1, &d, 1);
    axpy(nv, 0.75f, dx, dy);
    check("axpy");
    dump("axpy.y", 1, dy, nv);
    /* CSR SpMV, three spellings */
    int nr = 5000, nc = 4500;
    int* rowptr = malloc(sizeof(int) * (nr + 1));
    rowptr[0] = 0;
    for (int i = 0; i < nr; i++) rowptr[i + 1] = rowptr[i] + (int)(lcg() % (i % 97 == 0 ? 300 : 24));
    int nnz = rowptr[nr];
    int* col = malloc(sizeof(int) * nnz);
    float* val = fvec(nnz);
    for (int k = 0; k < nnz; k++) col[k] = (int)(lcg() % (uint32_t)nc);
    float *sx = fvec(nc), *s1 = calloc(nr, 4), *s2 = calloc(nr, 4), *s3 = calloc(nr, 4);
    dump("spmv.rowptr", 0, rowptr, nr + 1); dump("spmv.col", 0, col, nnz); dump("spmv.val", 1, val, nnz);
    dump("spmv.x", 1, sx, nc);
    spmv_vec(nr, nc, nnz, rowptr, col, val, sx, s1);
    check("spmv_vec");
    spmv_inline(nr, nc, nnz, rowptr, col, val, sx, s2);
    check("spmv_inline");
    spmv(nr, nc, nnz, rowptr, col, val, sx, s3);
    check("spmv");
    dump("spmv_vec.y", 1, s1, nr); dump("spmv_inline.y", 1, s2, nr); dump("spmv.y", 1, s3, nr);
    /* 5x5 stencils */
    int h = 61, w = 68;
    int* img = malloc(sizeof(int) * h * w);
    for (int i = 0; i < h * w; i++) img[i] = (int)(lcg() & 255);
    int k25[25], sharp[25];
    const int b5[5] = {1, 4, 6, 4, 1};
    for (int i = 0; i < 25; i++) {
        k25[i] = b5[i / 5] * b5[i % 5];
        sharp[i] = (int)(lcg() % 11) - 5;
    }
    int *o1 = calloc(h * w, 4), *o2 = calloc(h * w, 4);
    dump("conv.img", 0, img, h * w);
    conv5x5_u8(h, w, 256, img, k25, o1);
    check("conv5x5_u8");
    conv5x5_u8(h, w, 3, img, sharp, o2);
    check("conv5x5_u8 sharp");
    dump("conv.u8", 0, o1, h * w); dump("conv.u8s", 0, o2, h * w);
    float *fimg = fvec((long)h * w), *fk = fvec(25), *fo = fvec((long)h * w);
    dump("convf.o0", 1, fo, h * w);
    conv5x5_f32(h, w, fimg, fk, fo);
    check("conv5x5_f32");
    dump("convf.img", 1, fimg, h * w); dump("convf.k", 1, fk, 25); dump("convf.out", 1, fo, h * w);
    /* gemm */
    int gm = 64, gn = 48, gk = 40;
    float *gA = fvec((long)gm * gk), *gB = fvec((long)gk * gn), *gC = fvec((long)gm * gn);
    dump("gemm.A", 1, gA, (long)gm * gk); dump("gemm.B", 1, gB, (long)gk * gn); dump("gemm.C0", 1, gC, (long)gm * gn);
    gemm(gm, gn, gk, 1.0f, 0.5f, gA, gB, gC);
    check("gemm");
    dump("gemm.C", 1, gC, (long)gm * gn);
    fclose(out);
    return 0;
}
