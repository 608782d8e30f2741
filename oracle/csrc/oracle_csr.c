/* Plain, single-threaded CSR kernels for the CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library.  Shares no code with the CUDA path.
 *
 * Compiled with -O2 -ffp-contract=off: each product and sum is rounded separately,
 * in row order, exactly as the definition y_i = sum_p val[p] * x[col[p]] reads.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

/* y = M x, M in CSR (int64 rowptr, int32 col, double val). */
void oracle_csr_matvec(int64_t nrows, const int64_t *rowptr, const int32_t *col, const double *val,
                       const double *x, double *y) {
  for (int64_t i = 0; i < nrows; ++i) {
    double s = 0.0;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s += val[p] * x[col[p]];
    y[i] = s;
  }
}

/* Transpose: given M (nrows x ncols) in CSR, fill Mt (ncols x nrows) in CSR.
 * t_rowptr has ncols+1 entries; within each row of Mt the entries appear in
 * increasing original-row order (counting sort).  Returns 0, or -1 on bad input. */
int oracle_csr_transpose(int64_t nrows, int64_t ncols, const int64_t *rowptr, const int32_t *col,
                         const double *val, int64_t *t_rowptr, int32_t *t_col, double *t_val) {
  int64_t nnz = rowptr[nrows];
  memset(t_rowptr, 0, sizeof(int64_t) * (size_t)(ncols + 1));
  for (int64_t p = 0; p < nnz; ++p) {
    if (col[p] < 0 || col[p] >= ncols) return -1;
    t_rowptr[col[p] + 1] += 1;
  }
  for (int64_t j = 0; j < ncols; ++j) t_rowptr[j + 1] += t_rowptr[j];
  int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncols > 0 ? ncols : 1));
  if (!next) return -2;
  memcpy(next, t_rowptr, sizeof(int64_t) * (size_t)ncols);
  for (int64_t i = 0; i < nrows; ++i) {
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      int64_t q = next[col[p]]++;
      t_col[q] = (int32_t)i;
      t_val[q] = val[p];
    }
  }
  free(next);
  return 0;
}
