/*
 * Plain-C restatement of two elementary-order kernels -- TEST INFRASTRUCTURE
 * ONLY (oracle/__init__.py).  Built by oracle/cproj.py (gcc, -ffp-contract=off:
 * the compiler must not fuse the reference's separately rounded multiply and
 * subtract).
 *
 * cproj_project_f32  Step 3 of the sweep in the reference's order
 *                    (pkg/src/sketch_krylov/kernels.py:171-209 via
 *                    rbgs.py:369-370): acc = fl32(W); for l ascending:
 *                    acc = fl32(acc - fl32(fl32(Q[:,l]) * fl32(X[l,:]))).
 *                    Same arithmetic as oracle/sweep.py::gemm_ordered, which
 *                    the golden vectors pin; used where the numpy loop is too
 *                    slow (the 2^20-row kernel tests).
 * cproj_trsm_right   X = B R^{-1} row by row in binary64, l ascending with
 *                    fused multiply-adds, x_j = t * (1 / R_jj): the order of
 *                    the device's tall right solve (csrc/tri_const.cuh,
 *                    tri_solve_row) -- a bit-level check of the kernel's
 *                    own order at scale; the reference's (LAPACK dtrsm,
 *                    kernels.py:250-270) is checked with a tolerance.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

void cproj_project_f32(int64_t n, int c, int p, const float* Q, int64_t ldq, const double* X, int64_t ldx,
                       const float* W, int64_t ldw, float* out, int64_t ldo) {
  float* xs = (float*)malloc(sizeof(float) * (size_t)(c > 0 ? c : 1) * (size_t)p);
  for (int l = 0; l < c; ++l)
    for (int j = 0; j < p; ++j) xs[(int64_t)l * p + j] = (float)X[l + (int64_t)j * ldx];
#pragma omp parallel for schedule(static)
  for (int64_t r0 = 0; r0 < n; r0 += 64) {
    const int64_t r1 = r0 + 64 < n ? r0 + 64 : n;
    float acc[64][64];
    for (int64_t r = r0; r < r1; ++r)
      for (int j = 0; j < p; ++j) acc[r - r0][j] = W[r + (int64_t)j * ldw];
    for (int l = 0; l < c; ++l) {
      const float* xl = xs + (int64_t)l * p;
      const float* ql = Q + (int64_t)l * ldq;
      for (int64_t r = r0; r < r1; ++r) {
        const float q = ql[r];
        float* a = acc[r - r0];
        for (int j = 0; j < p; ++j) {
          const float t = q * xl[j];
          a[j] = a[j] - t;
        }
      }
    }
    for (int64_t r = r0; r < r1; ++r)
      for (int j = 0; j < p; ++j) out[r + (int64_t)j * ldo] = acc[r - r0][j];
  }
  free(xs);
}

void cproj_trsm_right(int64_t n, int p, const double* B, int64_t ldb, const double* R, int64_t ldr, double* out,
                      int64_t ldo) {
  double inv[64];
  for (int j = 0; j < p; ++j) inv[j] = 1.0 / R[j + (int64_t)j * ldr];
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    double x[64];
    for (int j = 0; j < p; ++j) x[j] = B[r + (int64_t)j * ldb];
    for (int j = 0; j < p; ++j) {
      double t = x[j];
      for (int l = 0; l < j; ++l) t = fma(-x[l], R[l + (int64_t)j * ldr], t);
      x[j] = t * inv[j];
    }
    for (int j = 0; j < p; ++j) out[r + (int64_t)j * ldo] = x[j];
  }
}
