/* C = alpha * A B + beta * C, all row-major. */
void gemm(int m, int n, int k, float alpha, float beta, float A[restrict const static m * k],
          float B[restrict const static k * n], float C[restrict const static m * n])
{
  #pragma pencil independent
  for (int i = 0; i < m; i++) {
    #pragma pencil independent
    for (int j = 0; j < n; j++) {
      float s;
      s = 0.0;
      #pragma pencil reduction (+: s)
      for (int p = 0; p < k; p++) {
        s += A[i * k + p] * B[p * n + j];
      }
      C[i * n + j] = alpha * s + beta * C[i * n + j];
    }
  }
}
