/* VOBLA transposed/strided view: y[j*incy] = alpha * sum_i A[i*lda + j] * x[i*incx] + beta * y[j*incy]. */
void gemv_t(int m, int n, int lda, int incx, int incy, float alpha, float beta,
            float A[restrict const static m * lda], float x[restrict const static m * incx],
            float y[restrict const static n * incy])
{
  #pragma pencil independent
  for (int j = 0; j < n; j++) {
    float s;
    s = 0.0;
    #pragma pencil reduction (+: s)
    for (int i = 0; i < m; i++) {
      s += A[i * lda + j] * x[i * incx];
    }
    y[j * incy] = alpha * s + beta * y[j * incy];
  }
}
