void axpy(int n, float a, float x[restrict const static n], float y[restrict const static n])
{
  for (int i = 0; i < n; i++) {
    y[i] = a * x[i] + y[i];
  }
}
