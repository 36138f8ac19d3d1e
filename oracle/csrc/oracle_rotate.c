/* ORACLE (test infrastructure only): the reference's Hadamard rotation
 * `rotate(x, H, placement)` (hadamard.py:45-57) evaluated in the exact
 * arithmetic order of the reference's numpy/OpenBLAS dgemm on this image:
 * each output element is a sequential fused-multiply-add accumulation over
 * the inner index j = 0..dim-1 starting from 0.0.  (Measured: identical bits
 * to `x @ H` / `H @ x` on every sampled element, including tie cases.)
 * H[j][c] = (-1)^popcount(j & c) / sqrt(dim)   (hadamard.py:31-42). */
#include <math.h>
#include <stdint.h>

static double entry(int j, int c, double h) { return (__builtin_popcount((unsigned)(j & c)) & 1) ? -h : h; }

/* post: out[r][c] = sum_j x[r][j] * H[j][c];  x, out: [rows][dim] */
void oracle_rotate_post(const double* x, int64_t rows, int dim, double* out) {
  const double h = 1.0 / sqrt((double)dim);
  for (int64_t r = 0; r < rows; ++r)
    for (int c = 0; c < dim; ++c) {
      double acc = 0.0;
      for (int j = 0; j < dim; ++j) acc = fma(x[r * dim + j], entry(j, c, h), acc);
      out[r * dim + c] = acc;
    }
}

/* pre: out[r][c] = sum_j H[r][j] * x[j][c];  x, out: [dim][cols] */
void oracle_rotate_pre(const double* x, int dim, int64_t cols, double* out) {
  const double h = 1.0 / sqrt((double)dim);
  for (int r = 0; r < dim; ++r)
    for (int64_t c = 0; c < cols; ++c) {
      double acc = 0.0;
      for (int j = 0; j < dim; ++j) acc = fma(entry(r, j, h), x[j * cols + c], acc);
      out[r * cols + c] = acc;
    }
}
