float dot(int n, float x[restrict const static n], float y[restrict const static n])
{
  float s;
  s = 0.0;
  #pragma pencil reduction (+: s)
  for (int i = 0; i < n; i++) {
    s += x[i] * y[i];
  }
  return s;
}
