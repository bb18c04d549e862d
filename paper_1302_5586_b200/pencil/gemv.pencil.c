/* y = alpha * A x + beta * y, A row-major m x n (VOBLA gemv over a plain view). */
void gemv(int m, int n, float alpha, float beta, float A[restrict const static m * n],
          float x[restrict const static n], float y[restrict const static m])
{
  #pragma pencil independent
  for (int i = 0; i < m; i++) {
    float s;
    s = 0.0;
    #pragma pencil reduction (+: s)
    for (int j = 0; j < n; j++) {
      s += A[i * n + j] * x[j];
    }
    y[i] = alpha * s + beta * y[i];
  }
}
