/*
 * rbgs_b200.h -- C ABI of the B200-native RBGS hot path (libs rbgs_b200.so).
 *
 * The reference (`sketch_krylov`, pure Python) has no FFI layer: its
 * boundary is the Python API of `rbgs.py` / `sketching.py` / `krylov.py`.
 * Each entry point below replaces one numeric site of that API (SURVEY.md
 * section 2, "kernel sites" K1-K10); the citation on each names the
 * reference lines it stands in for.  The Python host layer
 * (`paper_2111_14641_b200/rbgs.py` etc.) mirrors the reference API and calls
 * these through ctypes; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - every matrix pointer is DEVICE memory, column-major, leading dimension
 *     in elements (ld >= rows);
 *   - `dtype` arguments take RB_F32 / RB_F64;
 *   - `row0` is the global index of local row 0 (row sharding: the sketch
 *     operators are keyed by global row, so shards compose by summation);
 *   - every call is asynchronous on `stream` (a cudaStream_t, NULL = legacy
 *     default stream) and never synchronises the host;
 *   - concurrency: the library keeps no per-call device state of its own
 *     except the constant-bank copy of R used by the tall right solves
 *     (rb_trsm_right, rb_project_trsm); calls of those two on different
 *     streams of one device are serialised with an event (not inside a
 *     stream capture: a captured graph must not replay concurrently with
 *     other streams' solves on its device).  `ws` scratch belongs to the
 *     call's stream: two streams must pass different workspaces;
 *   - return value: RB_OK, or a negative RB_E* code with a message in
 *     rb_last_error();  numerical failures (non-PD pivot) are reported
 *     through device-side `info` words, as LAPACK does;
 *   - reductions over rows are two-stage with a fixed grid, so results are
 *     bit-reproducible run to run on the same device.
 */
#ifndef RBGS_B200_H
#define RBGS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RB_OK 0
#define RB_EINVAL (-1)   /* bad argument or shape                        */
#define RB_ECUDA (-2)    /* CUDA launch / runtime error                  */
#define RB_EWS (-3)      /* workspace too small                          */

#define RB_F32 0
#define RB_F64 1

/* Step-3 arithmetic order in coarse mode */
#define RB_ORDER_REFERENCE 0  /* separately rounded multiply and subtract  */
#define RB_ORDER_FMA 1        /* fused multiply-subtract (not bit-exact)    */
#define RB_ORDER_REFERENCE_SCALAR 2  /* RB_ORDER_REFERENCE issued as scalar
                                        FMUL + FADD instead of the packed
                                        FFMA2(-0) + FADD2 pair: same bits,
                                        the cross-check of the packed form */
#define RB_ORDER_TC 3         /* tensor pipe: Q X as three tcgen05 kind::tf32
                                 products of the hi/lo split operands
                                 (3xTF32, fp32 accumulation), binary32-level
                                 accuracy, HBM-bound; not the reference order */

const char* rb_version(void);
const char* rb_last_error(void);
/* Number of kernels this process has launched through the library. */
unsigned long long rb_launch_count(void);
/* Bytes of device workspace the sketch / reduction calls below may use for
 * an n-row, ncols-column, k-row problem (upper bound). */
size_t rb_workspace_bytes(int64_t n, int ncols, int k);

/* ---- K3  Step 3 projection (rbgs.py:369-370 -> kernels.py:171-209) -------
 * Qp = fl(W - Q X) in the reference's elementary order: acc = fl_c(W); for
 * l = 0..c-1 ascending: acc = fl_c(acc - fl_c(fl_c(Q[:,l]) * fl_c(X[l,:]))),
 * every multiply and subtract separately rounded in the compute format
 * (coarse: binary32, fine: binary64; no FMA contraction).  c may be 0.
 * order = RB_ORDER_FMA (coarse only) fuses each multiply-subtract into one
 * rounding instead: faster, not bit-identical to the reference.
 * norms2 (may be NULL) receives { sum W^2, sum Qp^2 } over these rows in
 * fp64 (rbgs.py:373-374 before the square root).                         */
int rb_project(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p,
               const void* Q, int64_t ldq, const double* X, int64_t ldx,
               const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* norms2,
               void* ws, size_t ws_bytes, void* stream);

/* Step 3 of block i with Step 5 of block i-1 fused in front (one-shot
 * sweeps): Qf, the last pf columns of Q[:, :c] (= Q'_(i-1), in place),
 * first becomes fl(Q'_(i-1) Rf^{-1}) (rbgs.py:281-283 -> kernels.py:250-270,
 * right solve with the pf x pf upper Rf), then the projection runs on the
 * updated Q.  Bitwise equal to rb_trsm_right(Qf -> Qf) + rb_project.     */
int rb_project_trsm(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p,
                    const void* Q, int64_t ldq, const double* X, int64_t ldx,
                    const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* norms2,
                    void* Qf, int64_t ldqf, const double* Rf, int64_t ldrf, int pf,
                    void* ws, size_t ws_bytes, void* stream);

/* ---- K1/K2  sketches (sketching.py:140-155 and the north-star kinds) -----
 * out (k x ncols, fp64, col-major, ld ldo) = Theta[:, row0:row0+n] @ X,
 * summed in fp64.  accumulate != 0 adds into out instead of overwriting.  */

/* gaussian kind: materialise the table of q = rint(2048 g) (an int16 value;
 * Philox4x32-10 + Box-Muller) for global rows
 * row0 .. row0+nrows-1 as two byte planes, hi = q >> 8 (signed) and
 * lo = q & 255, tiled in 128 x 128 blocks (csrc/gauss_layout.cuh).
 * ldt (padded row count) % 128 == 0; the buffer holds
 * 2 * ceil(k/128) * 128 * ldt bytes, padding zeroed.                      */
int rb_gaussian_fill(uint64_t seed, int k, int64_t row0, int64_t nrows,
                     uint8_t* theta, int64_t ldt, void* stream);
/* The same table with the operator's entries on a coarser grid: bits = 16 is
 * rb_gaussian_fill; bits = 8 stores q = 256 q8, q8 = clamp(rint(32 g), +-127)
 * (the same normals g on the int8 grid 2^-5; Theta = q / (8192 sqrt(k))), so
 * the lo plane is zero and rb_sketch_gaussian[2] called with mode + 16 skips
 * it: half the table stream and half the tensor work.  An opt-in operator
 * (discretised gaussian with 255 levels), not the default.               */
int rb_gaussian_fill_bits(uint64_t seed, int k, int64_t row0, int64_t nrows,
                          uint8_t* theta, int64_t ldt, int bits, void* stream);
/* out = scale * (q @ X) (scale = 1 / (2048 sqrt(k)) gives Theta @ X).
 * mode 0 = auto (tensor pipe for binary32 X, fp64 CUDA cores for binary64),
 * 1 = fp64 CUDA cores (exact fp64 products), 2 = tensor pipe: tcgen05
 * kind::i8 on the exact byte split of q and of X's per-chunk fixed-point
 * form (sketch_tc.cu), six byte digits of X (2^-47 of each 16384-row
 * chunk's max: binary64-grade), 3 = the same with the lean CTA, 4 / 5 =
 * tensor pipe with four / three digits (2^-31 / 2^-23 of the chunk max; 2/3
 * and 1/2 of the tensor work) for inputs whose R tolerates the rounding.  */
int rb_sketch_gaussian(int x_dtype, int64_t n, int ncols, const void* X, int64_t ldx,
                       const uint8_t* theta, int64_t ldt, int k, double scale,
                       double* out, int64_t ldo, int accumulate, int mode,
                       void* ws, size_t ws_bytes, void* stream);
/* Two-input form: [out1 | out2] = scale * (q @ [X1 | X2]) in ONE pass over
 * the table (the sweep sketches [Q'_i | W_(i+1)] together, halving the q
 * traffic).  c1, c2 <= 64; c2 may be 0.                                   */
int rb_sketch_gaussian2(int x1_dtype, const void* X1, int64_t ldx1, int c1,
                        int x2_dtype, const void* X2, int64_t ldx2, int c2, int64_t n,
                        const uint8_t* theta, int64_t ldt, int k, double scale,
                        double* out1, int64_t ldo1, double* out2, int64_t ldo2,
                        int accumulate, int mode, void* ws, size_t ws_bytes, void* stream);
/* The pre-pass (chunk exponents + digit planes) of the SECOND input of a
 * paired call (c1 + c2 > 64) on its own, so a caller can run it early on
 * another stream -- the sweep encodes W_(i+1) beside block i's projection --
 * and hand the buffer to rb_sketch_gaussian2_pre, which then skips it.  Same
 * plane bytes as the fused call.  out: rb_gauss_prepass_bytes(n, c2, c1,
 * digits) bytes, 256-byte aligned; digits must match the later call's mode. */
size_t rb_gauss_prepass_bytes(int64_t n, int c, int c_partner, int digits);
int rb_gauss_prepass(int x_dtype, const void* X, int64_t ldx, int c, int c_partner, int64_t n, int digits,
                     void* out, size_t out_bytes, void* stream);
int rb_sketch_gaussian2_pre(int x1_dtype, const void* X1, int64_t ldx1, int c1,
                            int x2_dtype, const void* X2, int64_t ldx2, int c2, int64_t n,
                            const uint8_t* theta, int64_t ldt, int k, double scale,
                            double* out1, int64_t ldo1, double* out2, int64_t ldo2,
                            int accumulate, int mode, const void* pre2, void* ws, size_t ws_bytes, void* stream);
/* srht kind (sketching.py:129-137): signs as a bitmask over the GLOBAL
 * padded index space (bit i set <=> sign_diagonal[i] = -1), sample = the
 * k global sample indices, scale = 1/sqrt(k).  Rows >= n_valid (global)
 * are the zero padding.  row0 must be a multiple of 2048 unless n_pad <= 2048. */
int rb_sketch_srht(int x_dtype, int64_t n, int ncols, const void* X, int64_t ldx,
                   int64_t row0, int64_t n_pad, const uint32_t* sign_bits,
                   const int64_t* sample, int k, double scale,
                   double* out, int64_t ldo, int accumulate,
                   void* ws, size_t ws_bytes, void* stream);
/* sparse_sign kind: s = min(nnz, k) nonzeros +-1/sqrt(s) per column of
 * Theta, rows from the Philox word stream. */
int rb_sketch_sparse_sign(int x_dtype, int64_t n, int ncols, const void* X, int64_t ldx,
                          int64_t row0, uint64_t seed, int k, int nnz,
                          double* out, int64_t ldo, int accumulate,
                          void* ws, size_t ws_bytes, void* stream);
/* sparse_sign kind, table path: pre-bucketed per 1024-row tile (built once
 * per operator shard by rb_sparse_sign_table: offs int32[ntiles][k+1],
 * lists uint16[ntiles][1024 * min(nnz, k)], ntiles = ceil(nrows / 1024));
 * the per-call sketch streams X and the table with a fixed summation
 * order.  Same operator as rb_sketch_sparse_sign (no reference
 * counterpart: the kind is a north-star addition). */
int rb_sparse_sign_table(uint64_t seed, int k, int nnz, int64_t row0, int64_t nrows,
                         int32_t* offs, uint16_t* lists, void* stream);
int rb_sketch_sparse_sign_tab(int x_dtype, int64_t n, int ncols, const void* X, int64_t ldx,
                              const int32_t* offs, const uint16_t* lists, int k, int nnz,
                              double* out, int64_t ldo, int accumulate,
                              void* ws, size_t ws_bytes, void* stream);
/* rademacher kind (sketching.py:151-155): k x n sign bits (row r at
 * bits + r * ldb words, bit i set <=> sign -1), out = scale * S @ X. */
int rb_sketch_signs(int x_dtype, int64_t n, int ncols, const void* X, int64_t ldx,
                    const uint32_t* bits, int64_t ldb, int k, double scale,
                    double* out, int64_t ldo, int accumulate,
                    void* ws, size_t ws_bytes, void* stream);

/* ---- K5  tall triangular scaling (rbgs.py:284, kernels.py:250-270) ------
 * Xout = B R^{-1} (R p x p upper, fp64), each row solved in fp64 and
 * rounded to out_dtype.  In place (Xout == B, same dtype) is allowed.     */
int rb_trsm_right(int in_dtype, int out_dtype, int64_t n, int p, const void* B, int64_t ldb,
                  const double* R, int64_t ldr, void* Xout, int64_t ldx, void* stream);

/* ---- small fp64 kernels (Steps 2, 4-5, 7; rbgs.py:144-225, 267-290, 428-443)
 * All hand-written (csrc/kdim.cu, small.cu): no library GEMMs.
 * C = alpha op(A) B + beta C, fp64 (numpy's `@` in the reference's LS
 * solvers, kernels.py / rbgs.py:144-212), op = transpose when transA != 0;
 * transB must be 0.  Split over K into ws (summed in split order:
 * deterministic) when the tile grid alone cannot fill the GPU.            */
int rb_gemm_f64(int transA, int transB, int m, int n, int k, double alpha,
                const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                double* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);
/* binary32 C = alpha op(A) B + beta C with binary32 accumulation -- the
 * Step-2 solvers in unique-coarse mode (fine = COARSE), where the reference
 * runs them in float32 (rbgs.py:144-212, prec.dtype).                     */
int rb_gemm_f32(int transA, int transB, int m, int n, int k, float alpha,
                const float* A, int64_t lda, const float* B, int64_t ldb, float beta,
                float* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);
/* Certification sums (rbgs.py:428-443) in ONE cooperative launch:
 * out[0] = ||I - S^T S||_F^2, out[1] = ||P - S R||_F^2, out[2] = ||P||_F^2
 * for S, P (k x m) and R (m x m), fixed summation order.                 */
int rb_certify(int k, int m, const double* S, int64_t lds, const double* P, int64_t ldp,
               const double* R, int64_t ldr, double* out, void* ws, size_t ws_bytes, void* stream);
/* out[0..2] = sums of squares of three binary64 matrices (one launch; the
 * per-block finiteness words of P_i, S_i, R_ii -- rbgs.py:380-388 through
 * the reference's Matrix() checks).  ws: >= 256 bytes of the caller's
 * scratch (CTA partials and arrival counters; no device globals). */
int rb_sumsq3(int64_t m1, int n1, const double* A1, int64_t lda1,
              int64_t m2, int n2, const double* A2, int64_t lda2,
              int64_t m3, int n3, const double* A3, int64_t lda3, double* out,
              void* ws, size_t ws_bytes, void* stream);
/* Symmetric rank-k update: C = alpha A^T A + beta C for a tall binary64 A
 * (k x n, C n x n; the upper triangle is valid: 128 x 64 tiles wholly below
 * the diagonal are not formed) -- the basis Gram of the
 * GMRES conditioning history (krylov.py:98-103, 247-257). */
int rb_syrk_f64(int n, int64_t k, double alpha, const double* A, int64_t lda, double beta,
                double* C, int64_t ldc, void* ws, size_t ws_bytes, void* stream);
/* Tall Gram / cross product: out (p x q fp64) = A^T B for n-row A (n x p)
 * and B (n x q), inputs f32 or f64, fp64 accumulation (fused l2 stage).  */
int rb_cross(int a_dtype, int b_dtype, int64_t n, int p, int q, const void* A, int64_t lda,
             const void* B, int64_t ldb, double* out, int64_t ldo, int accumulate,
             void* ws, size_t ws_bytes, void* stream);
/* Upper Cholesky R^T R = G (dpotrf, kernels.py:234-247); *info (device) =
 * 0 or the 1-based column of the first non-positive pivot.  R's strictly
 * lower part is zeroed.  G and R may alias.  p <= 1024.                  */
int rb_potrf_upper(int p, const double* G, int64_t ldg, double* R, int64_t ldr,
                   int* info, void* stream);
/* R factor (p x p upper, diag >= 0) of the Householder QR of a tall A (n x p,
 * p <= 64, binary32 or binary64; kernels.py:216-231 householder_qr, the l2
 * stage of rbgs.py:293-302) by sequential TSQR in binary64 -- backward
 * stable for any cond(A).  cond: when non-NULL and *cond == 0 on the device
 * the call does nothing (the sweep issues it behind the Gram Cholesky's
 * status word: no host branch).  info (may alias cond): 0 on a valid factor,
 * else the 1-based index of a zero / non-finite diagonal entry.
 * ws >= 2 * SMs * p * p doubles.                                          */
int rb_tsqr_r(int a_dtype, int64_t n, int p, const void* A, int64_t lda, double* R, int64_t ldr,
              const int* cond, int* info, void* ws, size_t ws_bytes, void* stream);
/* Left solve R X = B (R m x m upper), B m x nrhs overwritten with X.
 * *info (device) = 0, or 1 + index of the first zero diagonal.          */
int rb_trsm_left_upper(int m, int nrhs, const double* R, int64_t ldr, double* B, int64_t ldb,
                       int* info, void* stream);
/* Economic Householder QR of A (m x q, m >= q, fp64, overwritten by the
 * explicit Q) with R (q x q upper) and diag(R) >= 0 (kernels.py:216-231).
 * Single CTA; for the k-dimensional and Hessenberg problems only.        */
int rb_geqrf_small(int m, int q, double* A, int64_t lda, double* R, int64_t ldr,
                   void* ws, size_t ws_bytes, void* stream);
/* Sum of squares of an m x n fp64/f32 matrix, minus the identity when
 * minus_identity != 0 (certify, rbgs.py:441-442); result written (not
 * accumulated) to *out.                                                   */
int rb_sumsq(int dtype, int64_t m, int n, const void* A, int64_t lda, int minus_identity,
             double* out, void* ws, size_t ws_bytes, void* stream);

/* ---- composite Step-2 / Step-4-5 solvers ---------------------------------
 * Richardson (rbgs.py:144-156): X (c x p) after l sweeps of
 * X <- X + S^T (P - S X) from X = 0.  T is a k x p fp64 scratch.  ONE
 * cooperative launch (grid barriers between the split-K GEMM phases).
 * p <= 64.                                                               */
int rb_ls_richardson(int k, int c, int p, const double* S, int64_t lds, const double* P,
                     int64_t ldp, int l, double* X, int64_t ldx, double* T, int64_t ldt,
                     void* ws, size_t ws_bytes, void* stream);
/* One sketched-CholQR pass on the k x p sketch Sp (rbgs.py:282-289):
 * G = Sp^T Sp, R = chol(G) (info as rb_potrf_upper), Sout = Sp R^{-1}
 * (rows solved in rb_trsm_right's order).  ONE cooperative launch.       */
int rb_sketched_cholqr_small(int k, int p, const double* Sp, int64_t lds, double* R,
                             int64_t ldr, double* Sout, int64_t ldso, int* info,
                             void* ws, size_t ws_bytes, void* stream);

/* l2_plus_cholqr without a host branch (rbgs.py:293-302): given both
 * outcomes of the Gram stage -- (A) R_a, S_a from R' = chol(Q'^T Q') and the
 * sketched CholQR of Q' R'^{-1}, (B) R_b, S_b from the one-pass sketched
 * CholQR of Q' -- keep A when *info_sel == 0 (R' existed), else B: R (p x p),
 * S (k x p) and *info_out = the kept path's Cholesky info.              */
int rb_l2_select(int k, int p, const int* info_sel, const int* info_a, const int* info_b,
                 const double* Ra, int64_t ldra, const double* Sa, int64_t ldsa,
                 const double* Rb, int64_t ldrb, const double* Sb, int64_t ldsb,
                 double* R, int64_t ldr, double* S, int64_t lds, int* info_out, void* stream);

/* ---- K10  operator: 7-point Dirichlet Laplacian (C4, krylov.py:129-130) --
 * Y = A X on an nx*ny*nz_local slab (x fastest) of the global grid; halo
 * planes (nx*ny rows each, NULL = Dirichlet boundary) supply the z
 * neighbours of the first / last local plane.                             */
int rb_stencil7(int x_dtype, int y_dtype, int nx, int ny, int nz_local, int ncols,
                const void* X, int64_t ldx, const void* halo_lo, const void* halo_hi,
                int64_t ldh, void* Y, int64_t ldy, void* stream);

/* General CSR operator (operators.py:57-73): Y = A X, A n x n CSR with
 * int64 indptr / indices and fp64 values; each output row accumulates its
 * entries in stored order from 0 (scipy csr_matvecs order).             */
int rb_csr_spmm(int x_dtype, int y_dtype, int64_t n, int ncols, const int64_t* indptr,
                const int64_t* indices, const double* values, const void* X, int64_t ldx,
                void* Y, int64_t ldy, void* stream);

/* ---- misc ---------------------------------------------------------------- */
/* Y = (out dtype) X elementwise for an m x n matrix (rounding to nearest). */
int rb_convert(int in_dtype, int out_dtype, int64_t m, int n, const void* X, int64_t ldx,
               void* Y, int64_t ldy, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RBGS_B200_H */
