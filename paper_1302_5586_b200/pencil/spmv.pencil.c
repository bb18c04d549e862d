/* CSR sparse matrix-vector product, three PENCIL spellings of the same nest:
   spmv_vec    - independent row loop, licensed reduction over the row (reassociation allowed)
   spmv_inline - independent row loop, row sum in source order
   spmv        - row loop over a call whose irregular gather is described by an ACCESS summary */
void spmv_vec(int nrows, int ncols, int nnz, int rowptr[restrict const static nrows + 1],
              int col[restrict const static nnz], float val[restrict const static nnz],
              float x[restrict const static ncols], float y[restrict const static nrows])
{
  #pragma pencil independent
  for (int i = 0; i < nrows; i++) {
    float s;
    s = 0.0;
    #pragma pencil reduction (+: s)
    for (int k = rowptr[i]; k < rowptr[i + 1]; k++) {
      s += val[k] * x[col[k]];
    }
    y[i] = s;
  }
}

void spmv_inline(int nrows, int ncols, int nnz, int rowptr[restrict const static nrows + 1],
                 int col[restrict const static nnz], float val[restrict const static nnz],
                 float x[restrict const static ncols], float y[restrict const static nrows])
{
  #pragma pencil independent
  for (int i = 0; i < nrows; i++) {
    float s;
    s = 0.0;
    for (int k = rowptr[i]; k < rowptr[i + 1]; k++) {
      s += val[k] * x[col[k]];
    }
    y[i] = s;
  }
}

void spmv_row_summary(int nrows, int ncols, int nnz, int i,
                      int rowptr[restrict const static nrows + 1],
                      int col[restrict const static nnz], float val[restrict const static nnz],
                      float x[restrict const static ncols], float y[restrict const static nrows])
{
  USE(rowptr[i]);
  USE(rowptr[i + 1]);
  for (int k = 0; k < nnz; k++) {
    USE(col[k]);
    USE(val[k]);
  }
  for (int j = 0; j < ncols; j++) {
    USE(x[j]);
  }
  DEF(y[i]);
}

void spmv_row(int nrows, int ncols, int nnz, int i, int rowptr[restrict const static nrows + 1],
              int col[restrict const static nnz], float val[restrict const static nnz],
              float x[restrict const static ncols], float y[restrict const static nrows])
    ACCESS(spmv_row_summary(nrows, ncols, nnz, i, rowptr, col, val, x, y))
{
  float s;
  s = 0.0;
  for (int k = rowptr[i]; k < rowptr[i + 1]; k++) {
    s += val[k] * x[col[k]];
  }
  y[i] = s;
}

void spmv(int nrows, int ncols, int nnz, int rowptr[restrict const static nrows + 1],
          int col[restrict const static nnz], float val[restrict const static nnz],
          float x[restrict const static ncols], float y[restrict const static nrows])
{
  for (int i = 0; i < nrows; i++) {
    spmv_row(nrows, ncols, nnz, i, rowptr, col, val, x, y);
  }
}
