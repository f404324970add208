// extern "C" boundary of librbgs_b200.so (include/rbgs_b200.h).
#include <stdarg.h>

#include <mutex>

#include "common.cuh"

namespace rb {

static thread_local char g_err[512] = "";
unsigned long long g_launches = 0;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return RB_ECUDA;
  }
  return RB_OK;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

int project(int, int, int, int, int64_t, int, int, const void*, int64_t, const double*, int64_t, const void*, int64_t,
            void*, int64_t, double*, void*, size_t, cudaStream_t);
int project_trsm(int, int, int, int, int64_t, int, int, const void*, int64_t, const double*, int64_t, const void*,
                 int64_t, void*, int64_t, double*, void*, int64_t, const double*, int64_t, int, void*, size_t,
                 cudaStream_t);
int gaussian_fill(uint64_t, int, int64_t, int64_t, uint8_t*, int64_t, cudaStream_t, int bits);
int sketch_gaussian(int, int64_t, int, const void*, int64_t, const uint8_t*, int64_t, int, double, double*, int64_t,
                    int, int, void*, size_t, cudaStream_t);
size_t gauss_tc_ws_bytes(int64_t n, int ncols, int k);
int sketch_gaussian2(int, const void*, int64_t, int, int, const void*, int64_t, int, int64_t, const uint8_t*, int64_t,
                     int, double, double*, int64_t, double*, int64_t, int, int, void*, size_t, cudaStream_t,
                     const void* pre2);
size_t gauss_prepass_bytes(int64_t n, int c, int c_partner, int dig);
int gauss_prepass(int, const void*, int64_t, int, int, int64_t, int, void*, size_t, cudaStream_t);
int sketch_signs(int, int64_t, int, const void*, int64_t, const uint32_t*, int64_t, int, double, double*, int64_t, int,
                 void*, size_t, cudaStream_t);
int sketch_srht(int, int64_t, int, const void*, int64_t, int64_t, int64_t, const uint32_t*, const int64_t*, int,
                double, double*, int64_t, int, void*, size_t, cudaStream_t);
int sketch_sparse_sign(int, int64_t, int, const void*, int64_t, int64_t, uint64_t, int, int, double*, int64_t, int,
                       void*, size_t, cudaStream_t);
int sparse_sign_table(uint64_t, int, int, int64_t, int64_t, int32_t*, uint16_t*, cudaStream_t);
int sketch_sparse_sign_tab(int, int64_t, int, const void*, int64_t, const int32_t*, const uint16_t*, int, int, double*,
                           int64_t, int, void*, size_t, cudaStream_t);
int trsm_right(int, int, int64_t, int, const void*, int64_t, const double*, int64_t, void*, int64_t, cudaStream_t);
int gemm_f64(int, int, int, int, int, double, const double*, int64_t, const double*, int64_t, double, double*,
             int64_t, void*, size_t, cudaStream_t);
int cross(int, int, int64_t, int, int, const void*, int64_t, const void*, int64_t, double*, int64_t, int, void*,
          size_t, cudaStream_t);
int syrk_f64(int, int64_t, double, const double*, int64_t, double, double*, int64_t, void*, size_t, cudaStream_t);
int sumsq3(int64_t, int, const double*, int64_t, int64_t, int, const double*, int64_t, int64_t, int, const double*,
           int64_t, double*, void*, size_t, cudaStream_t);
int gemm_f32(int, int, int, int, int, float, const float*, int64_t, const float*, int64_t, float, float*, int64_t,
             void*, size_t, cudaStream_t);
int certify(int, int, const double*, int64_t, const double*, int64_t, const double*, int64_t, double*, void*, size_t,
            cudaStream_t);
size_t kdim_ws_bytes(int k, int m);
int l2_select(int, int, const int*, const int*, const int*, const double*, int64_t, const double*, int64_t,
              const double*, int64_t, const double*, int64_t, double*, int64_t, double*, int64_t, int*, cudaStream_t);
int potrf_upper(int, const double*, int64_t, double*, int64_t, int*, cudaStream_t);
int tsqr_r(int, int64_t, int, const void*, int64_t, double*, int64_t, const int*, int*, void*, size_t, cudaStream_t);
int trsm_left_upper(int, int, const double*, int64_t, double*, int64_t, int*, cudaStream_t);
int geqrf_small(int, int, double*, int64_t, double*, int64_t, void*, size_t, cudaStream_t);
int sumsq(int, int64_t, int, const void*, int64_t, int, double*, void*, size_t, cudaStream_t);
int ls_richardson(int, int, int, const double*, int64_t, const double*, int64_t, int, double*, int64_t, double*,
                  int64_t, void*, size_t, cudaStream_t);
int sketched_cholqr_small(int, int, const double*, int64_t, double*, int64_t, double*, int64_t, int*, void*, size_t,
                          cudaStream_t);
int stencil7(int, int, int, int, int, int, const void*, int64_t, const void*, const void*, int64_t, void*, int64_t,
             cudaStream_t);
int convert(int, int, int64_t, int, const void*, int64_t, void*, int64_t, cudaStream_t);
int csr_spmm(int, int, int64_t, int, const int64_t*, const int64_t*, const double*, const void*, int64_t, void*,
             int64_t, cudaStream_t);

}  // namespace rb

using rb::as_stream;

extern "C" {

const char* rb_version(void) { return "rbgs_b200 0.1.0 (sm_100a)"; }
const char* rb_last_error(void) { return rb::g_err; }
unsigned long long rb_launch_count(void) { return rb::g_launches; }

size_t rb_workspace_bytes(int64_t n, int ncols, int k) {
  // Split-K partials are bounded by ~4 waves of (128 x 64) fp64 tiles; the
  // per-CTA norm partials by n / 256 pairs; a single-split gemm by k x ncols.
  const size_t kk = (size_t)(k > 64 ? k : 64), cc = (size_t)(ncols > 64 ? ncols : 64);
  const size_t tiles = (size_t)8 * rb::sm_count() * 128 * 64 * sizeof(double);
  const size_t norms = ((size_t)(n > 0 ? n : 0) / 128 + 64) * 2 * sizeof(double);
  const size_t single = kk * cc * sizeof(double) * 2;
  size_t b = tiles > norms ? tiles : norms;
  b = b > single ? b : single;
  const size_t g = rb::gauss_tc_ws_bytes(n, ncols, k);
  b = b > g ? b : g;
  const size_t kd = rb::kdim_ws_bytes(k, ncols > k ? ncols : k);
  return (b > kd ? b : kd) + (1u << 20);
}

int rb_project(int qd, int wd, int cd, int order, int64_t n, int c, int p, const void* Q, int64_t ldq,
               const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* norms2,
               void* ws, size_t wsb, void* s) {
  return rb::project(qd, wd, cd, order, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, norms2, ws, wsb, as_stream(s));
}

int rb_project_trsm(int qd, int wd, int cd, int order, int64_t n, int c, int p, const void* Q, int64_t ldq,
                    const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* norms2,
                    void* Qf, int64_t ldqf, const double* Rf, int64_t ldrf, int pf, void* ws, size_t wsb, void* s) {
  return rb::project_trsm(qd, wd, cd, order, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, norms2, Qf, ldqf, Rf, ldrf,
                          pf, ws, wsb, as_stream(s));
}

int rb_gaussian_fill(uint64_t seed, int k, int64_t row0, int64_t nrows, uint8_t* theta, int64_t ldt, void* s) {
  return rb::gaussian_fill(seed, k, row0, nrows, theta, ldt, as_stream(s), 16);
}

int rb_gaussian_fill_bits(uint64_t seed, int k, int64_t row0, int64_t nrows, uint8_t* theta, int64_t ldt, int bits,
                          void* s) {
  return rb::gaussian_fill(seed, k, row0, nrows, theta, ldt, as_stream(s), bits);
}

int rb_sketch_gaussian(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const uint8_t* theta, int64_t ldt,
                       int k, double scale, double* out, int64_t ldo, int acc, int mode, void* ws, size_t wsb,
                       void* s) {
  return rb::sketch_gaussian(xd, n, ncols, X, ldx, theta, ldt, k, scale, out, ldo, acc, mode, ws, wsb, as_stream(s));
}

int rb_sketch_gaussian2(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                        int64_t n, const uint8_t* theta, int64_t ldt, int k, double scale, double* out1, int64_t ldo1,
                        double* out2, int64_t ldo2, int acc, int mode, void* ws, size_t wsb, void* s) {
  return rb::sketch_gaussian2(xd1, X1, ld1, c1, xd2, X2, ld2, c2, n, theta, ldt, k, scale, out1, ldo1, out2, ldo2, acc,
                              mode, ws, wsb, as_stream(s), nullptr);
}

int rb_sketch_gaussian2_pre(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                            int64_t n, const uint8_t* theta, int64_t ldt, int k, double scale, double* out1,
                            int64_t ldo1, double* out2, int64_t ldo2, int acc, int mode, const void* pre2, void* ws,
                            size_t wsb, void* s) {
  return rb::sketch_gaussian2(xd1, X1, ld1, c1, xd2, X2, ld2, c2, n, theta, ldt, k, scale, out1, ldo1, out2, ldo2, acc,
                              mode, ws, wsb, as_stream(s), pre2);
}

size_t rb_gauss_prepass_bytes(int64_t n, int c, int c_partner, int digits) {
  return rb::gauss_prepass_bytes(n, c, c_partner, digits);
}

int rb_gauss_prepass(int xd, const void* X, int64_t ldx, int c, int c_partner, int64_t n, int digits, void* out,
                     size_t out_bytes, void* s) {
  return rb::gauss_prepass(xd, X, ldx, c, c_partner, n, digits, out, out_bytes, as_stream(s));
}

int rb_sketch_srht(int xd, int64_t n, int ncols, const void* X, int64_t ldx, int64_t row0, int64_t n_pad,
                   const uint32_t* bits, const int64_t* sample, int k, double scale, double* out, int64_t ldo,
                   int acc, void* ws, size_t wsb, void* s) {
  return rb::sketch_srht(xd, n, ncols, X, ldx, row0, n_pad, bits, sample, k, scale, out, ldo, acc, ws, wsb,
                         as_stream(s));
}

int rb_sketch_sparse_sign(int xd, int64_t n, int ncols, const void* X, int64_t ldx, int64_t row0, uint64_t seed,
                          int k, int nnz, double* out, int64_t ldo, int acc, void* ws, size_t wsb, void* s) {
  return rb::sketch_sparse_sign(xd, n, ncols, X, ldx, row0, seed, k, nnz, out, ldo, acc, ws, wsb, as_stream(s));
}

int rb_sparse_sign_table(uint64_t seed, int k, int nnz, int64_t row0, int64_t nrows, int32_t* offs, uint16_t* lists,
                         void* s) {
  return rb::sparse_sign_table(seed, k, nnz, row0, nrows, offs, lists, as_stream(s));
}

int rb_sketch_sparse_sign_tab(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const int32_t* offs,
                              const uint16_t* lists, int k, int nnz, double* out, int64_t ldo, int acc, void* ws,
                              size_t wsb, void* s) {
  return rb::sketch_sparse_sign_tab(xd, n, ncols, X, ldx, offs, lists, k, nnz, out, ldo, acc, ws, wsb, as_stream(s));
}

int rb_sketch_signs(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const uint32_t* bits, int64_t ldb,
                    int k, double scale, double* out, int64_t ldo, int acc, void* ws, size_t wsb, void* s) {
  return rb::sketch_signs(xd, n, ncols, X, ldx, bits, ldb, k, scale, out, ldo, acc, ws, wsb, as_stream(s));
}

int rb_trsm_right(int ind, int outd, int64_t n, int p, const void* B, int64_t ldb, const double* R, int64_t ldr,
                  void* X, int64_t ldx, void* s) {
  return rb::trsm_right(ind, outd, n, p, B, ldb, R, ldr, X, ldx, as_stream(s));
}

int rb_gemm_f32(int tA, int tB, int m, int n, int k, float alpha, const float* A, int64_t lda, const float* B,
                int64_t ldb, float beta, float* C, int64_t ldc, void* ws, size_t wsb, void* s) {
  return rb::gemm_f32(tA, tB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, wsb, as_stream(s));
}

int rb_l2_select(int k, int p, const int* info_sel, const int* info_a, const int* info_b, const double* Ra,
                 int64_t ldra, const double* Sa, int64_t ldsa, const double* Rb, int64_t ldrb, const double* Sb,
                 int64_t ldsb, double* R, int64_t ldr, double* S, int64_t lds, int* info_out, void* s) {
  return rb::l2_select(k, p, info_sel, info_a, info_b, Ra, ldra, Sa, ldsa, Rb, ldrb, Sb, ldsb, R, ldr, S, lds,
                       info_out, as_stream(s));
}

int rb_certify(int k, int m, const double* S, int64_t lds, const double* P, int64_t ldp, const double* R,
               int64_t ldr, double* out, void* ws, size_t wsb, void* s) {
  return rb::certify(k, m, S, lds, P, ldp, R, ldr, out, ws, wsb, as_stream(s));
}

int rb_gemm_f64(int tA, int tB, int m, int n, int k, double alpha, const double* A, int64_t lda, const double* B,
                int64_t ldb, double beta, double* C, int64_t ldc, void* ws, size_t wsb, void* s) {
  return rb::gemm_f64(tA, tB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, wsb, as_stream(s));
}

int rb_sumsq3(int64_t m1, int n1, const double* A1, int64_t lda1, int64_t m2, int n2, const double* A2, int64_t lda2,
              int64_t m3, int n3, const double* A3, int64_t lda3, double* out, void* ws, size_t wsb, void* s) {
  return rb::sumsq3(m1, n1, A1, lda1, m2, n2, A2, lda2, m3, n3, A3, lda3, out, ws, wsb, as_stream(s));
}

int rb_syrk_f64(int n, int64_t k, double alpha, const double* A, int64_t lda, double beta, double* C, int64_t ldc,
                void* ws, size_t wsb, void* s) {
  return rb::syrk_f64(n, k, alpha, A, lda, beta, C, ldc, ws, wsb, as_stream(s));
}

int rb_cross(int ad, int bd, int64_t n, int p, int q, const void* A, int64_t lda, const void* B, int64_t ldb,
             double* out, int64_t ldo, int acc, void* ws, size_t wsb, void* s) {
  return rb::cross(ad, bd, n, p, q, A, lda, B, ldb, out, ldo, acc, ws, wsb, as_stream(s));
}

int rb_potrf_upper(int p, const double* G, int64_t ldg, double* R, int64_t ldr, int* info, void* s) {
  return rb::potrf_upper(p, G, ldg, R, ldr, info, as_stream(s));
}

int rb_tsqr_r(int ad, int64_t n, int p, const void* A, int64_t lda, double* R, int64_t ldr, const int* cond, int* info,
              void* ws, size_t wsb, void* s) {
  return rb::tsqr_r(ad, n, p, A, lda, R, ldr, cond, info, ws, wsb, as_stream(s));
}

int rb_trsm_left_upper(int m, int nrhs, const double* R, int64_t ldr, double* B, int64_t ldb, int* info, void* s) {
  return rb::trsm_left_upper(m, nrhs, R, ldr, B, ldb, info, as_stream(s));
}

int rb_geqrf_small(int m, int q, double* A, int64_t lda, double* R, int64_t ldr, void* ws, size_t wsb, void* s) {
  return rb::geqrf_small(m, q, A, lda, R, ldr, ws, wsb, as_stream(s));
}

int rb_sumsq(int dt, int64_t m, int n, const void* A, int64_t lda, int minus_id, double* out, void* ws, size_t wsb,
             void* s) {
  return rb::sumsq(dt, m, n, A, lda, minus_id, out, ws, wsb, as_stream(s));
}

int rb_ls_richardson(int k, int c, int p, const double* S, int64_t lds, const double* P, int64_t ldp, int l,
                     double* X, int64_t ldx, double* T, int64_t ldt, void* ws, size_t wsb, void* s) {
  return rb::ls_richardson(k, c, p, S, lds, P, ldp, l, X, ldx, T, ldt, ws, wsb, as_stream(s));
}

int rb_sketched_cholqr_small(int k, int p, const double* Sp, int64_t lds, double* R, int64_t ldr, double* Sout,
                             int64_t ldso, int* info, void* ws, size_t wsb, void* s) {
  return rb::sketched_cholqr_small(k, p, Sp, lds, R, ldr, Sout, ldso, info, ws, wsb, as_stream(s));
}

int rb_stencil7(int xd, int yd, int nx, int ny, int nzl, int ncols, const void* X, int64_t ldx, const void* hlo,
                const void* hhi, int64_t ldh, void* Y, int64_t ldy, void* s) {
  return rb::stencil7(xd, yd, nx, ny, nzl, ncols, X, ldx, hlo, hhi, ldh, Y, ldy, as_stream(s));
}

int rb_convert(int ind, int outd, int64_t m, int n, const void* X, int64_t ldx, void* Y, int64_t ldy, void* s) {
  return rb::convert(ind, outd, m, n, X, ldx, Y, ldy, as_stream(s));
}

int rb_csr_spmm(int xd, int yd, int64_t n, int ncols, const int64_t* indptr, const int64_t* indices,
                const double* vals, const void* X, int64_t ldx, void* Y, int64_t ldy, void* s) {
  return rb::csr_spmm(xd, yd, n, ncols, indptr, indices, vals, X, ldx, Y, ldy, as_stream(s));
}

}  // extern "C"
