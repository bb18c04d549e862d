/* Synthetic inputs for the bench and tests.
 *
 * One 64-bit LCG stream per config — the constants of the reference interpreter's
 * `rand` fallback (interp.cpp:249-253): s <- s*6364136223846793005 + 1442695040888963407,
 * r = s >> 33.  Draw t (t >= 1) is the state after t steps from the seed.
 *   fp32 value  = (r & 0xffffff) / 2^24 - 0.5        (uniform [-0.5, 0.5), exact in fp32)
 *   u8 value    = r & 255
 *   column idx  = r % ncols
 * Streams are generated in parallel: every OpenMP chunk jumps ahead to its first draw
 * (affine-map doubling), so the output is independent of the thread count.
 *
 * Host-only utility (no CUDA): not on the kernel path, shared by bench.py's two arms.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LCG_A 6364136223846793005ull
#define LCG_C 1442695040888963407ull

/* state after `steps` steps from s */
static uint64_t lcg_jump(uint64_t s, uint64_t steps) {
    uint64_t a = LCG_A, c = LCG_C, ra = 1, rc = 0;
    while (steps) {
        if (steps & 1) { ra = ra * a; rc = rc * a + c; }
        c = c * a + c;
        a = a * a;
        steps >>= 1;
    }
    return ra * s + rc;
}
static inline uint64_t lcg_next(uint64_t* s) {
    *s = *s * LCG_A + LCG_C;
    return *s >> 33;
}
static inline float r_to_f32(uint64_t r) {
    return (float)(r & 0xffffffu) * (1.0f / 16777216.0f) - 0.5f;
}

#define CHUNK (1ll << 16)

/* out[i] = fp32 value of draw (first + i + 1) */
void pencil_synth_f32(float* out, long long n, unsigned long long seed, long long first) {
#pragma omp parallel for schedule(static)
    for (long long c0 = 0; c0 < n; c0 += CHUNK) {
        uint64_t s = lcg_jump(seed, (uint64_t)(first + c0));
        long long e = c0 + CHUNK < n ? c0 + CHUNK : n;
        for (long long i = c0; i < e; i++) out[i] = r_to_f32(lcg_next(&s));
    }
}

/* out[i] = (draw & 255) as int32 (u8 image held in int, the PENCIL drop-in layout) */
void pencil_synth_u8_i32(int* out, long long n, unsigned long long seed, long long first) {
#pragma omp parallel for schedule(static)
    for (long long c0 = 0; c0 < n; c0 += CHUNK) {
        uint64_t s = lcg_jump(seed, (uint64_t)(first + c0));
        long long e = c0 + CHUNK < n ? c0 + CHUNK : n;
        for (long long i = c0; i < e; i++) out[i] = (int)(lcg_next(&s) & 255u);
    }
}

/* out[i] = draw & 255 as bytes (packed u8 image) */
void pencil_synth_u8(unsigned char* out, long long n, unsigned long long seed, long long first) {
#pragma omp parallel for schedule(static)
    for (long long c0 = 0; c0 < n; c0 += CHUNK) {
        uint64_t s = lcg_jump(seed, (uint64_t)(first + c0));
        long long e = c0 + CHUNK < n ? c0 + CHUNK : n;
        for (long long i = c0; i < e; i++) out[i] = (unsigned char)(lcg_next(&s) & 255u);
    }
}

/* ---- power-law CSR (SURVEY §8d SpMV config) ----------------------------------------
 * Row length len_i = min(maxlen, max(1, floor(xm * u_i^(-1/alpha)))), u_i = ((r & 0xffffff) + 0.5)/2^24
 * from draws 1..nrows; xm is bisected so sum(len) is as close as possible to
 * avg_per_row * nrows.  Then, row by row, draws (nrows + 2k + 1, nrows + 2k + 2) give
 * col[k] = r % ncols and val[k]; columns are sorted within each row (val follows).
 *
 * Phase 1 fills rowptr[0..nrows] and returns nnz (or -1 if it exceeds INT32 range);
 * phase 2 fills col/val for the caller-allocated nnz arrays. */
long long pencil_synth_csr_rowptr(int nrows, double avg_per_row, double alpha, int maxlen,
                                  unsigned long long seed, int* rowptr, double* xm_out) {
    double* v = (double*)malloc(sizeof(double) * (size_t)(nrows > 0 ? nrows : 1));
    if (!v) return -2;
#pragma omp parallel for schedule(static)
    for (long long c0 = 0; c0 < nrows; c0 += CHUNK) {
        uint64_t s = lcg_jump(seed, (uint64_t)c0);
        long long e = c0 + CHUNK < nrows ? c0 + CHUNK : nrows;
        for (long long i = c0; i < e; i++) {
            double u = ((double)(lcg_next(&s) & 0xffffffu) + 0.5) / 16777216.0;
            v[i] = pow(u, -1.0 / alpha);
        }
    }
    double target = avg_per_row * (double)nrows;
    double lo = 1e-6, hi = avg_per_row * 4.0 + 1.0, best = hi, best_err = 1e300;
    for (int it = 0; it < 80; it++) {
        double xm = 0.5 * (lo + hi);
        long long tot = 0;
#pragma omp parallel for reduction(+ : tot) schedule(static)
        for (long long i = 0; i < nrows; i++) {
            double l = floor(xm * v[i]);
            long long li = l < 1.0 ? 1 : (l > (double)maxlen ? maxlen : (long long)l);
            tot += li;
        }
        double err = fabs((double)tot - target);
        if (err < best_err) { best_err = err; best = xm; }
        if ((double)tot < target) lo = xm; else hi = xm;
    }
    long long nnz = 0;
    rowptr[0] = 0;
    for (long long i = 0; i < nrows; i++) {
        double l = floor(best * v[i]);
        long long li = l < 1.0 ? 1 : (l > (double)maxlen ? maxlen : (long long)l);
        nnz += li;
        if (nnz > 2147483647ll) { free(v); return -1; }
        rowptr[i + 1] = (int)nnz;
    }
    free(v);
    if (xm_out) *xm_out = best;
    return nnz;
}

static void sort_row(int* c, float* v, long long n) {
    if (n < 2) return;
    if (n <= 32) {
        for (long long a = 1; a < n; a++) {
            int kc = c[a];
            float kv = v[a];
            long long b = a - 1;
            while (b >= 0 && c[b] > kc) { c[b + 1] = c[b]; v[b + 1] = v[b]; b--; }
            c[b + 1] = kc;
            v[b + 1] = kv;
        }
        return;
    }
    /* in-place heap sort on (c, v) pairs: no allocation, O(n log n) */
    for (long long start = n / 2 - 1; start >= 0; start--) {
        long long root = start;
        for (;;) {
            long long ch = 2 * root + 1;
            if (ch >= n) break;
            if (ch + 1 < n && c[ch] < c[ch + 1]) ch++;
            if (c[root] >= c[ch]) break;
            int tc = c[root]; c[root] = c[ch]; c[ch] = tc;
            float tv = v[root]; v[root] = v[ch]; v[ch] = tv;
            root = ch;
        }
    }
    for (long long end = n - 1; end > 0; end--) {
        int tc = c[0]; c[0] = c[end]; c[end] = tc;
        float tv = v[0]; v[0] = v[end]; v[end] = tv;
        long long root = 0;
        for (;;) {
            long long ch = 2 * root + 1;
            if (ch >= end) break;
            if (ch + 1 < end && c[ch] < c[ch + 1]) ch++;
            if (c[root] >= c[ch]) break;
            tc = c[root]; c[root] = c[ch]; c[ch] = tc;
            tv = v[root]; v[root] = v[ch]; v[ch] = tv;
            root = ch;
        }
    }
}

void pencil_synth_csr_fill(int nrows, int ncols, unsigned long long seed, const int* rowptr,
                           int* col, float* val) {
    const long long RCH = 4096;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long r0 = 0; r0 < nrows; r0 += RCH) {
        long long r1 = r0 + RCH < nrows ? r0 + RCH : nrows;
        uint64_t s = lcg_jump(seed, (uint64_t)nrows + 2ull * (uint64_t)rowptr[r0]);
        for (long long k = rowptr[r0]; k < rowptr[r1]; k++) {
            col[k] = (int)(lcg_next(&s) % (uint64_t)ncols);
            val[k] = r_to_f32(lcg_next(&s));
        }
        for (long long i = r0; i < r1; i++)
            sort_row(col + rowptr[i], val + rowptr[i], (long long)rowptr[i + 1] - rowptr[i]);
    }
}
