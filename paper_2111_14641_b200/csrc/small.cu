// Small fp64 kernels for the k- and m-dimensional steps of the sweep:
// Step 2 (rbgs.py:144-225), the sketched Cholesky-QR (rbgs.py:267-290),
// certification (rbgs.py:428-443), the tall triangular scaling of Steps 4-5
// (rbgs.py:284, kernels.py:250-270) and the Householder QR used by the
// direct LS solver and the GMRES least-squares problem (kernels.py:216-231).
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "tri_const.cuh"

namespace rb {

int sm_count();

namespace {

constexpr int kThreads = 256;

// ============================ generic GEMM ==================================
// C = alpha op(A) op(B) + beta C; fp64 accumulation, split-K over a fixed
// grid (deterministic).  A, B may be binary32 (promoted on load).
constexpr int GBM = 64, GBN = 64, GBK = 16;

template <typename TA, typename TB>
__global__ void __launch_bounds__(kThreads)
gemm_partial(int tA, int tB, int m, int n, int64_t k, const TA* __restrict__ A, int64_t lda,
             const TB* __restrict__ B, int64_t ldb, int64_t chunk, double* __restrict__ ws) {
  __shared__ __align__(16) double sA[GBK][GBM];
  __shared__ __align__(16) double sB[GBK][GBN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.x * GBM, n0 = blockIdx.y * GBN;
  const int64_t kb = (int64_t)blockIdx.z * chunk, ke = min(k, kb + chunk);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += GBK) {
    __syncthreads();
    for (int e = threadIdx.x; e < GBM * GBK; e += kThreads) {
      int i, kk;
      if (tA) { kk = e % GBK; i = e / GBK; } else { i = e % GBM; kk = e / GBM; }
      const int64_t kg = k0 + kk;
      double v = 0.0;
      if (m0 + i < m && kg < ke) v = tA ? (double)A[kg + (int64_t)(m0 + i) * lda] : (double)A[(m0 + i) + kg * lda];
      sA[kk][i] = v;
    }
    for (int e = threadIdx.x; e < GBN * GBK; e += kThreads) {
      int j, kk;
      if (tB) { j = e % GBN; kk = e / GBN; } else { kk = e % GBK; j = e / GBK; }
      const int64_t kg = k0 + kk;
      double v = 0.0;
      if (n0 + j < n && kg < ke) v = tB ? (double)B[(n0 + j) + kg * ldb] : (double)B[kg + (int64_t)(n0 + j) * ldb];
      sB[kk][j] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) a[q] = sA[kk][ty + 16 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) b[q] = sB[kk][tx + 16 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[q][t] = fma(a[q], b[t], acc[q][t]);
    }
  }
  double* dst = ws + (int64_t)blockIdx.z * m * n;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = m0 + ty + 16 * q, j = n0 + tx + 16 * t;
      if (i < m && j < n) dst[i + (int64_t)j * m] = acc[q][t];
    }
}

__global__ void gemm_epilogue(const double* __restrict__ ws, int splits, int m, int n, double alpha,
                              double beta, double* __restrict__ C, int64_t ldc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)m * n;
  if (e >= tot) return;
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += ws[(int64_t)q * tot + e];
  const int i = (int)(e % m), j = (int)(e / m);
  double* c = C + i + (int64_t)j * ldc;
  *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
}

template <typename TA, typename TB>
int gemm_t(int tA, int tB, int m, int n, int64_t k, double alpha, const TA* A, int64_t lda,
           const TB* B, int64_t ldb, double beta, double* C, int64_t ldc, void* ws,
           size_t wsb, cudaStream_t st) {
  if (m == 0 || n == 0) return RB_OK;
  const int mt = ceil_div(m, GBM), nt = ceil_div(n, GBN);
  const size_t per = (size_t)m * n * sizeof(double);
  int64_t splits = std::max<int64_t>(1, std::min<int64_t>((k + 255) / 256, (4 * sm_count() + mt * nt - 1) / (mt * nt)));
  if ((size_t)splits * per > wsb) splits = std::max<int64_t>(1, (int64_t)(wsb / per));
  RB_REQUIRE(ws && (size_t)splits * per <= wsb, "gemm: workspace too small (%zu B for %d x %d)", per, m, n);
  RB_REQUIRE(splits <= 65535, "gemm: too many splits");
  int64_t chunk = k > 0 ? (k + splits - 1) / splits : 0;
  chunk = (chunk + GBK - 1) / GBK * GBK;
  splits = chunk > 0 ? (k + chunk - 1) / chunk : 0;
  if (splits > 0)
    RB_KLAUNCH gemm_partial<TA, TB><<<dim3(mt, nt, (unsigned)splits), kThreads, 0, st>>>(tA, tB, m, n, k, A, lda, B, ldb, chunk,
                                                                                 (double*)ws);
  RB_KLAUNCH gemm_epilogue<<<ceil_div((int64_t)m * n, 256), 256, 0, st>>>((double*)ws, (int)splits, m, n, alpha, beta, C, ldc);
  return check_launch("gemm");
}

// ============================ Cholesky ======================================
// Right-looking, upper, in shared memory (p <= 128) -- dpotrf semantics:
// info = j (1-based) at the first pivot that is <= 0 or NaN.
__global__ void potrf_kernel(int p, const double* __restrict__ G, int64_t ldg, double* __restrict__ R,
                             int64_t ldr, int* __restrict__ info) {
  extern __shared__ double S[];  // p x p column-major
  __shared__ int bad;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e % p, j = e / p;
    S[e] = (i <= j) ? G[i + (int64_t)j * ldg] : 0.0;
  }
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double d = S[j + j * p];
    if (!(d > 0.0)) {  // catches NaN too
      if (threadIdx.x == 0) bad = j + 1;
      break;
    }
    const double r = sqrt(d);
    // scale row j right of the diagonal (every thread has read d: the
    // diagonal is only rewritten after the next barrier)
    for (int c = j + 1 + threadIdx.x; c < p; c += blockDim.x) S[j + c * p] /= r;
    __syncthreads();
    if (threadIdx.x == 0) S[j + j * p] = r;
    // trailing update of the upper part: S[a, b] -= S[j, a] S[j, b],
    // j < a <= b; lanes along a (column-contiguous), warps along b
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
    for (int b = j + 1 + ty; b < p; b += ny) {
      const double sjb = S[j + b * p];
      for (int a = j + 1 + tx; a <= b; a += 32) S[a + b * p] -= S[j + a * p] * sjb;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e % p, j = e / p;
    R[i + (int64_t)j * ldr] = (i <= j) ? S[e] : 0.0;
  }
  if (threadIdx.x == 0) *info = bad;
}

// ============================ triangular solves =============================
// Tall right solve X = B R^{-1} by forward substitution in fp64, one row per
// thread in registers, l ascending (dot form); R and 1 / R_jj come from the
// constant bank (tri_const.cuh: the shared-memory version was bound by the
// per-lane register writeback of its broadcast loads).
template <typename TI, typename TO, int PB, int RPT>
__global__ void __launch_bounds__(kThreads, 2)  // 2 CTAs/SM even at p = 64 (a few spills beat 8 warps/SM)
trsm_right_kernel(int64_t n, int p, const TI* B, int64_t ldb, TO* Xo, int64_t ldx) {  // B, Xo may alias
  static_assert(RPT == 1, "one row per thread");
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) x[j] = j < p ? (double)B[r + (int64_t)j * ldb] : 0.0;
  tri_solve_row<PB, (PB <= 40 ? 4 : 2)>(x, p);
#pragma unroll
  for (int j = 0; j < PB; ++j)
    if (j < p) Xo[r + (int64_t)j * ldx] = (TO)x[j];
}

// More than 40 columns: `x[64]` in binary64 is 128 registers and spilled
// (4.97 ms at 2^24 x 64).  Here the first 32 solved entries of the row stay
// in registers and the later ones go to shared memory ([l - 32][thread],
// conflict-free), columns 32.. solved four at a time as independent chains.
// Every column keeps the reference chain -- s = x_j; s = fma(-x_l, R_lj, s)
// for l ascending; x_j = s / R_jj (as s * (1 / R_jj), like tri_solve_row) --
// so the output is bitwise that of trsm_right_kernel.
constexpr int kTrsmHiThreads = 256;
template <typename TI, typename TO, int PB>
__global__ void __launch_bounds__(kTrsmHiThreads, 2)
trsm_right_hi_kernel(int64_t n, int p, const TI* B, int64_t ldb, TO* Xo, int64_t ldx) {  // B, Xo may alias
  static_assert(PB > 32 && PB <= 64 && PB % 4 == 0, "columns 33 .. 64");
  extern __shared__ double trsm_sh[];  // [PB - 32][kTrsmHiThreads]
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double* xh = trsm_sh + threadIdx.x;
  double x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (double)B[r + (int64_t)j * ldb];  // p > 32 here
  tri_solve_row<32, 4>(x, 32);
#pragma unroll
  for (int j = 0; j < 32; ++j) Xo[r + (int64_t)j * ldx] = (TO)x[j];
#pragma unroll
  for (int j = 32; j < PB; j += 4) {
    if (j >= p) break;
    double s[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) s[c] = j + c < p ? (double)B[r + (int64_t)(j + c) * ldb] : 0.0;
#pragma unroll
    for (int l = 0; l < 32; ++l)
#pragma unroll
      for (int c = 0; c < 4; ++c) s[c] = fma(-x[l], c_tri_R[l + (j + c) * kTriLd], s[c]);
#pragma unroll
    for (int l = 32; l < j; ++l) {
      const double xl = xh[(l - 32) * kTrsmHiThreads];
#pragma unroll
      for (int c = 0; c < 4; ++c) s[c] = fma(-xl, c_tri_R[l + (j + c) * kTriLd], s[c]);
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (j + c < p) {
        const double xj = s[c] * c_tri_inv[j + c];
        xh[(j + c - 32) * kTrsmHiThreads] = xj;
        Xo[r + (int64_t)(j + c) * ldx] = (TO)xj;
#pragma unroll
        for (int c2 = c + 1; c2 < 4; ++c2) s[c2] = fma(-xj, c_tri_R[j + c + (j + c2) * kTriLd], s[c2]);
      }
    }
  }
}

// Left solve R X = B in place, one warp per right-hand side.
__global__ void trsm_left_upper_kernel(int m, int nrhs, const double* __restrict__ R, int64_t ldr,
                                       double* __restrict__ B, int64_t ldb, int* __restrict__ info) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int bad = 0;
    for (int i = 0; i < m; ++i)
      if (R[i + (int64_t)i * ldr] == 0.0) { bad = i + 1; break; }
    *info = bad;
  }
  if (warp >= nrhs) return;
  double* b = B + (int64_t)warp * ldb;
  for (int i = m - 1; i >= 0; --i) {
    double s = 0.0;
    for (int l = i + 1 + lane; l < m; l += 32) s += R[i + (int64_t)l * ldr] * b[l];
    s = warp_sum(s);
    if (lane == 0) b[i] = (b[i] - s) / R[i + (int64_t)i * ldr];
    __syncwarp();
  }
}

// ============================ Householder QR (single CTA) ===================
// A (m x q) -> explicit economic Q in A, R (q x q) with diag(R) >= 0.
// Workspace: V (m x q) reflectors + tau (q).
__global__ void __launch_bounds__(1024)
geqrf_kernel(int m, int q, double* __restrict__ A, int64_t lda, double* __restrict__ R, int64_t ldr,
             double* __restrict__ V, double* __restrict__ tau) {
  __shared__ double red[32];
  __shared__ double sh[4];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  auto bsum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    return s;
  };
  for (int j = 0; j < q; ++j) {
    double s = 0.0;
    for (int i = j + 1 + tid; i < m; i += nt) { const double a = A[i + (int64_t)j * lda]; s += a * a; }
    const double tail2 = bsum(s);
    const double alpha = A[j + (int64_t)j * lda];
    const double nrm = sqrt(tail2 + alpha * alpha);
    // v = x - beta e1 with beta = -sign(alpha) ||x||, unit-normalised; H = I - 2 v v^T
    const double beta = alpha >= 0.0 ? -nrm : nrm;  // R_jj before the sign fix
    const double v0 = alpha - beta;
    const double vn2 = tail2 + v0 * v0;
    const bool skip = !(nrm > 0.0) || !(vn2 > 0.0);
    for (int i = tid; i < m; i += nt) {
      double v = 0.0;
      if (!skip && i >= j) v = (i == j ? v0 : A[i + (int64_t)j * lda]) / sqrt(vn2);
      V[i + (int64_t)j * m] = v;
    }
    if (tid == 0) tau[j] = skip ? 0.0 : 2.0;
    __syncthreads();
    // apply H = I - tau v v^T to the trailing columns, one warp per column
    if (!skip) {
      for (int c = j + 1 + warp; c < q; c += nw) {
        double d = 0.0;
        for (int i = j + lane; i < m; i += 32) d += V[i + (int64_t)j * m] * A[i + (int64_t)c * lda];
        d = warp_sum(d) * 2.0;
        for (int i = j + lane; i < m; i += 32) A[i + (int64_t)c * lda] -= d * V[i + (int64_t)j * m];
      }
    }
    __syncthreads();
    if (tid == 0) sh[0] = skip ? alpha : beta;
    __syncthreads();
    // column j of R: rows < j already final in A, diagonal = beta
    for (int i = tid; i < q; i += nt) {
      double v = 0.0;
      if (i < j) v = A[i + (int64_t)j * lda];
      else if (i == j) v = sh[0];
      R[i + (int64_t)j * ldr] = v;
    }
    __syncthreads();
  }
  // explicit Q: start from [I; 0], apply H_{q-1} .. H_0
  for (int e = tid; e < m * q; e += nt) {
    const int i = e % m, c = e / m;
    A[i + (int64_t)c * lda] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = q - 1; j >= 0; --j) {
    if (tau[j] != 0.0) {
      for (int c = j + warp; c < q; c += nw) {
        double d = 0.0;
        for (int i = j + lane; i < m; i += 32) d += V[i + (int64_t)j * m] * A[i + (int64_t)c * lda];
        d = warp_sum(d) * 2.0;
        for (int i = j + lane; i < m; i += 32) A[i + (int64_t)c * lda] -= d * V[i + (int64_t)j * m];
      }
    }
    __syncthreads();
  }
  // sign fix: diag(R) >= 0 (zero stays zero)
  __shared__ signed char neg[1024];
  for (int c = tid; c < q; c += nt) neg[c] = R[c + (int64_t)c * ldr] < 0.0;
  __syncthreads();
  for (int e = tid; e < m * q; e += nt) {
    const int c = e / m;
    if (neg[c]) A[(e % m) + (int64_t)c * lda] = -A[(e % m) + (int64_t)c * lda];
  }
  for (int e = tid; e < q * q; e += nt) {
    const int i = e % q, c = e / q;
    if (i > c) R[i + (int64_t)c * ldr] = 0.0;
    else if (neg[i]) R[i + (int64_t)c * ldr] = -R[i + (int64_t)c * ldr];
  }
}

// ============================ sum of squares ================================
template <typename T>
__global__ void sumsq_partial(int64_t m, int n, const T* __restrict__ A, int64_t lda, int minus_id,
                              double* __restrict__ part) {
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  const int64_t tot = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    double v = (double)A[i + j * lda];
    if (minus_id && i == j) v = 1.0 - v;
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_vec(const double* __restrict__ part, int count, double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double s = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

template <typename TI, typename TO>
__global__ void convert_kernel(int64_t m, int n, const TI* __restrict__ X, int64_t ldx, TO* __restrict__ Y,
                               int64_t ldy) {
  const int64_t tot = m * n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % m, j = e / m;
    Y[i + j * ldy] = (TO)X[i + j * ldx];
  }
}

__global__ void copy_f64(int m, int n, const double* __restrict__ A, int64_t lda, double* __restrict__ B,
                         int64_t ldb) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * n) return;
  const int i = (int)(e % m), j = (int)(e / m);
  B[i + (int64_t)j * ldb] = A[i + (int64_t)j * lda];
}

template <typename TI, typename TO>
void trsm_right_launch(int64_t n, int p, const void* B, int64_t ldb, const double* R, int64_t ldr, void* X,
                       int64_t ldx, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(tri_mutex());
  if (load_tri_const_locked(p, R, ldr, st) != RB_OK) return;
#define RB_TR(V)                                                                                          \
  if (p <= V) {                                                                                           \
    constexpr int RPT = 1;                                                                                \
    RB_KLAUNCH trsm_right_kernel<TI, TO, V, RPT><<<ceil_div(n, (int64_t)RPT * kThreads), kThreads, 0, st>>>( \
        n, p, (const TI*)B, ldb, (TO*)X, ldx);                                                            \
    tri_const_done_locked(st);                                                                            \
    return;                                                                                               \
  }
  RB_TR(4) RB_TR(8) RB_TR(12) RB_TR(16) RB_TR(24) RB_TR(32) RB_TR(40)
  static const int hi = getenv("RB_TRSM_HI") ? atoi(getenv("RB_TRSM_HI")) : 1;
  if (hi) {
#define RB_TRH(V)                                                                                              \
  if (p <= V) {                                                                                                \
    const size_t smem = (size_t)(V - 32) * kTrsmHiThreads * sizeof(double);                                    \
    cudaFuncSetAttribute(trsm_right_hi_kernel<TI, TO, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                         (int)smem);                                                                           \
    RB_KLAUNCH trsm_right_hi_kernel<TI, TO, V><<<ceil_div(n, (int64_t)kTrsmHiThreads), kTrsmHiThreads, smem,   \
                                                 st>>>(n, p, (const TI*)B, ldb, (TO*)X, ldx);                  \
    tri_const_done_locked(st);                                                                                 \
    return;                                                                                                    \
  }
    RB_TRH(48) RB_TRH(64)
#undef RB_TRH
  }
  RB_TR(48) RB_TR(64)
#undef RB_TR
}

}  // namespace

// Tall-skinny cross product out = A^T B for p, q <= 8 (the l2 stage's
// Q'^T Q' at block width 4 / 8): the split-K tile kernel
// would multiply a 128 x 16 register tile of mostly padding per row.  Here
// a thread keeps the p x q products of its rows in registers, a CTA reduces
// them in a fixed order and writes one partial; the partials are summed in
// CTA order (deterministic).  HBM-bound: (p + q) s bytes per row.
template <typename TA, typename TB, int PB>
__global__ void __launch_bounds__(kThreads)
cross_small_partial(int64_t n, int p, int q, const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B,
                    int64_t ldb, int64_t rows_per_cta, double* __restrict__ ws) {
  __shared__ double red[kThreads / 32][PB * PB];
  double acc[PB][PB];
#pragma unroll
  for (int a = 0; a < PB; ++a)
#pragma unroll
    for (int b = 0; b < PB; ++b) acc[a][b] = 0.0;
  const int64_t beg = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t end = min(n, beg + rows_per_cta);
  for (int64_t i = beg + threadIdx.x; i < end; i += kThreads) {
    double x[PB], y[PB];
#pragma unroll
    for (int a = 0; a < PB; ++a) x[a] = a < p ? (double)A[i + (int64_t)a * lda] : 0.0;
#pragma unroll
    for (int b = 0; b < PB; ++b) y[b] = b < q ? (double)B[i + (int64_t)b * ldb] : 0.0;
#pragma unroll
    for (int a = 0; a < PB; ++a)
#pragma unroll
      for (int b = 0; b < PB; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int a = 0; a < PB; ++a)
#pragma unroll
    for (int b = 0; b < PB; ++b) {
      const double v = warp_sum(acc[a][b]);
      if (lane == 0) red[warp][a * PB + b] = v;
    }
  __syncthreads();
  for (int e = threadIdx.x; e < p * q; e += kThreads) {
    const int a = e % p, b = e / p;
    double v = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) v += red[w][a * PB + b];
    ws[(int64_t)blockIdx.x * p * q + e] = v;  // column-major p x q partial
  }
}

template <typename TA, typename TB>
int cross_small(int64_t n, int p, int q, const TA* A, int64_t lda, const TB* B, int64_t ldb, double beta,
                double* out, int64_t ldo, void* ws, size_t wsb, cudaStream_t st) {
  const size_t per = (size_t)p * q * sizeof(double);
  int ctas = (int)std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, 4 * sm_count()));
  if ((size_t)ctas * per > wsb) ctas = (int)std::max<size_t>(1, wsb / per);
  RB_REQUIRE(ws && (size_t)ctas * per <= wsb, "rb_cross: workspace too small");
  const int64_t rpc = (n + ctas - 1) / ctas;
  if (n > 0) {
    if (p <= 4 && q <= 4)
      RB_KLAUNCH cross_small_partial<TA, TB, 4><<<ctas, kThreads, 0, st>>>(n, p, q, A, lda, B, ldb, rpc, (double*)ws);
    else
      RB_KLAUNCH cross_small_partial<TA, TB, 8><<<ctas, kThreads, 0, st>>>(n, p, q, A, lda, B, ldb, rpc, (double*)ws);
  }
  RB_KLAUNCH gemm_epilogue<<<ceil_div((int64_t)p * q, 256), 256, 0, st>>>((double*)ws, n > 0 ? ctas : 0, p, q, 1.0,
                                                                       beta, out, ldo);
  return check_launch("rb_cross (small)");
}

// Tall cross product out = A^T B for 8 < max(p, q) <= 64 (the l2 stage's
// Q'^T Q' at block widths 16 .. 64, rbgs.py:293-302) on the FP64 tensor pipe:
// mma.sync m16n8k4 f64.  The split-K tile kernel above issued 8 scalar
// shared loads per 16 DFMA and padded a 40 x 40 output to 64 x 64 (0.95 ms
// per 1e6 x 40 block, 3.4 TFLOP/s).  Here a CTA walks its row range in
// 64-row chunks (coalesced column reads, staged as binary64 [column][row]
// with a pitch of 68: staging stores and fragment loads are conflict-free), a warp owns one 16-row tile of
// the output for a quarter / half of the chunk's rows and all its 8-column
// tiles (one A fragment per k-step serves every column tile); for a Gram
// (A == B) tiles wholly below the diagonal are skipped and mirrored by the
// reduction.  Fixed orders throughout: per-warp k ascending, warps, then
// CTAs in index order.
constexpr int kCrossKC = 64, kCrossPitch = 68, kCrossThreads = 256;

template <typename TA, typename TB>
__global__ void __launch_bounds__(kCrossThreads, 2)
cross_dmma_partial(int64_t n, int p, int q, const TA* __restrict__ A, int64_t lda, const TB* __restrict__ B,
                   int64_t ldb, int64_t rows_per_cta, int sym, double* __restrict__ ws) {
  extern __shared__ double cross_sm[];
  double* sA = cross_sm;                                  // [column][kCrossPitch]
  double* sB = sym ? sA : cross_sm + 64 * kCrossPitch;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int mt = (p + 15) / 16, nt = (q + 7) / 8;
  const int groups = 8 / mt;                              // k-groups (warps per output row tile)
  const int mtile = warp % mt, kg = warp / mt;
  const bool active = kg < groups;
  const int m0 = mtile * 16;
  const int kper = kCrossKC / groups;                     // rows of a chunk per k-group (multiple of 4)
  double acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  const int64_t beg = (int64_t)blockIdx.x * rows_per_cta, end = min(n, beg + rows_per_cta);
  for (int64_t r0 = beg; r0 < end; r0 += kCrossKC) {
    __syncthreads();
    // stage: lanes along rows (64 consecutive rows of one column per two warps' worth of lanes)
    for (int e = tid; e < kCrossKC * p; e += kCrossThreads) {
      const int kk = e % kCrossKC, j = e / kCrossKC;
      const int64_t r = r0 + kk;
      sA[j * kCrossPitch + kk] = r < end ? (double)A[r + (int64_t)j * lda] : 0.0;
    }
    if (!sym)
      for (int e = tid; e < kCrossKC * q; e += kCrossThreads) {
        const int kk = e % kCrossKC, j = e / kCrossKC;
        const int64_t r = r0 + kk;
        sB[j * kCrossPitch + kk] = r < end ? (double)B[r + (int64_t)j * ldb] : 0.0;
      }
    __syncthreads();
    if (active) {
      const int kb = kg * kper;
      for (int k0 = kb; k0 < kb + kper; k0 += 4) {
        const double a0 = (m0 + g < p) ? sA[(m0 + g) * kCrossPitch + k0 + t] : 0.0;
        const double a1 = (m0 + g + 8 < p) ? sA[(m0 + g + 8) * kCrossPitch + k0 + t] : 0.0;
#pragma unroll
        for (int nn = 0; nn < 8; ++nn) {
          if (nn < nt && !(sym && 8 * (nn + 1) <= m0)) {
            const int col = nn * 8 + g;
            const double b0 = col < q ? sB[col * kCrossPitch + k0 + t] : 0.0;
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(acc[nn][0]), "+d"(acc[nn][1]), "+d"(acc[nn][2]), "+d"(acc[nn][3])
                         : "d"(a0), "d"(a1), "d"(b0));
          }
        }
      }
    }
  }
  // CTA reduction over the k-groups in group order (through shared memory)
  __syncthreads();
  double* red = cross_sm;  // [groups][16 mt x 64], reuses the staging area (sized by the launcher)
  const size_t gstride = (size_t)16 * mt * 64;
  if (active) {
#pragma unroll
    for (int nn = 0; nn < 8; ++nn) {
      if (nn < nt) {
        const int c0 = nn * 8 + 2 * t;
        double* d = red + (size_t)kg * gstride;
        d[(m0 + g) * 64 + c0] = acc[nn][0];
        d[(m0 + g) * 64 + c0 + 1] = acc[nn][1];
        d[(m0 + g + 8) * 64 + c0] = acc[nn][2];
        d[(m0 + g + 8) * 64 + c0 + 1] = acc[nn][3];
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < p * q; e += kCrossThreads) {
    const int i = e % p, j = e / p;
    double v = 0.0;
    for (int w = 0; w < groups; ++w) v += red[(size_t)w * gstride + i * 64 + j];
    ws[(int64_t)blockIdx.x * p * q + e] = v;  // column-major p x q partial
  }
}

__global__ void cross_dmma_reduce(const double* __restrict__ ws, int parts, int p, int q, int sym, double beta,
                                  double* __restrict__ out, int64_t ldo) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= p * q) return;
  const int i = e % p, j = e / p;
  if (sym && i > j) return;  // written by (j, i)
  double v = 0.0;
  for (int c = 0; c < parts; ++c) v += ws[(int64_t)c * p * q + e];
  double* o = out + i + (int64_t)j * ldo;
  *o = beta == 0.0 ? v : v + beta * *o;
  if (sym && i < j) {
    double* o2 = out + j + (int64_t)i * ldo;
    *o2 = beta == 0.0 ? v : v + beta * *o2;
  }
}

template <typename TA, typename TB>
int cross_dmma(int64_t n, int p, int q, const TA* A, int64_t lda, const TB* B, int64_t ldb, double beta, double* out,
               int64_t ldo, void* ws, size_t wsb, cudaStream_t st) {
  const bool sym = (const void*)A == (const void*)B && p == q && lda == ldb && std::is_same<TA, TB>::value;
  const size_t per = (size_t)p * q * sizeof(double);
  int ctas = (int)std::min<int64_t>(2 * (int64_t)sm_count(), std::max<int64_t>(1, (n + kCrossKC - 1) / kCrossKC));
  if ((size_t)ctas * per > wsb) ctas = (int)std::max<size_t>(1, wsb / per);
  RB_REQUIRE(ws && (size_t)ctas * per <= wsb, "rb_cross: workspace too small");
  int64_t rows = (n + ctas - 1) / ctas;
  rows = (rows + kCrossKC - 1) / kCrossKC * kCrossKC;
  ctas = (int)std::max<int64_t>(1, (n + rows - 1) / rows);
  const int mt = (p + 15) / 16, groups = 8 / mt;
  const size_t stage = (size_t)(sym ? 1 : 2) * 64 * kCrossPitch * sizeof(double);
  const size_t smem = std::max(stage, (size_t)groups * 16 * mt * 64 * sizeof(double));
  cudaFuncSetAttribute(cross_dmma_partial<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  RB_KLAUNCH cross_dmma_partial<TA, TB><<<ctas, kCrossThreads, smem, st>>>(n, p, q, A, lda, B, ldb, rows, sym ? 1 : 0,
                                                                           (double*)ws);
  RB_KLAUNCH cross_dmma_reduce<<<ceil_div((int64_t)p * q, 256), 256, 0, st>>>((const double*)ws, ctas, p, q, sym ? 1 : 0,
                                                                              beta, out, ldo);
  return check_launch("rb_cross (dmma)");
}

int cross(int ad, int bd, int64_t n, int p, int q, const void* A, int64_t lda, const void* B, int64_t ldb,
          double* out, int64_t ldo, int acc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(n >= 0 && p >= 1 && q >= 1 && out && ldo >= p, "rb_cross: bad args");
  const double beta = acc ? 1.0 : 0.0;
  if (p <= 8 && q <= 8) {
    if (ad == RB_F32 && bd == RB_F32)
      return cross_small<float, float>(n, p, q, (const float*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
    if (ad == RB_F32)
      return cross_small<float, double>(n, p, q, (const float*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
    if (bd == RB_F32)
      return cross_small<double, float>(n, p, q, (const double*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
    return cross_small<double, double>(n, p, q, (const double*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
  }
  static const int use_dmma = getenv("RB_CROSS_DMMA") ? atoi(getenv("RB_CROSS_DMMA")) : 1;
  if (use_dmma && p <= 64 && q <= 64 && n > 0) {
    if (ad == RB_F32 && bd == RB_F32)
      return cross_dmma<float, float>(n, p, q, (const float*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
    if (ad == RB_F32)
      return cross_dmma<float, double>(n, p, q, (const float*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
    if (bd == RB_F32)
      return cross_dmma<double, float>(n, p, q, (const double*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
    return cross_dmma<double, double>(n, p, q, (const double*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
  }
  if (ad == RB_F32 && bd == RB_F32)
    return gemm_t<float, float>(1, 0, p, q, n, 1.0, (const float*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
  if (ad == RB_F32)
    return gemm_t<float, double>(1, 0, p, q, n, 1.0, (const float*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
  if (bd == RB_F32)
    return gemm_t<double, float>(1, 0, p, q, n, 1.0, (const double*)A, lda, (const float*)B, ldb, beta, out, ldo, ws, wsb, st);
  return gemm_t<double, double>(1, 0, p, q, n, 1.0, (const double*)A, lda, (const double*)B, ldb, beta, out, ldo, ws, wsb, st);
}

// ============================ tall QR, R factor only (TSQR) =================
// R (p x p, upper, diag >= 0) with A = Q R for a tall A (n x p, p <= 64), by
// Householder reflections in binary64 -- the l2 stage of l2_plus_cholqr
// (rbgs.py:293-302 -> kernels.householder_qr, kernels.py:216-231) when the
// Gram route Q'^T Q' = R'^T R' breaks down (cond(Q') > ~1e8): Householder
// stays backward stable for any conditioning, like the reference's LAPACK QR.
// Sequential TSQR: a CTA walks its row range in slabs of kTsRows - p rows,
// each time factoring [R_running; slab] (kTsRows x p, in shared memory) and
// keeping the new p x p R; the per-CTA factors are stacked and factored the
// same way by one CTA.  One row per thread; a reflector is applied to the
// trailing columns warp by warp (a warp owns a column: dot, then update --
// no block barrier inside a step beyond the two that publish the reflector).
// `cond`: when non-null and *cond == 0 the kernel returns at once -- the
// sweep launches it unconditionally behind the Gram Cholesky's status word,
// so there is no host branch and the common path costs two empty launches.
constexpr int kTsRows = 256, kTsThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kTsThreads)
tsqr_seq(int64_t n, int p, const T* __restrict__ A, int64_t lda, int64_t rows_per_cta, double* __restrict__ Rstack,
         int64_t lds, const int* __restrict__ cond, int final_fix, int* __restrict__ info_out) {
  if (cond && *cond == 0) return;
  extern __shared__ double ts_sm[];
  double* M = ts_sm;                    // [p][kTsRows] column-major tile
  double* red = ts_sm + (size_t)p * kTsRows;  // [8] warp partials + [2] scalars
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t beg = (int64_t)blockIdx.x * rows_per_cta, end = min(n, beg + rows_per_cta);
  const int slab = kTsRows - p;
  for (int c = 0; c < p; ++c) M[c * kTsRows + tid] = 0.0;  // running R = 0
  for (int64_t r0 = beg; r0 < end || r0 == beg; r0 += slab) {
    // rows p .. kTsRows-1 <- the slab (zero padded)
    if (tid >= p) {
      const int64_t r = r0 + (tid - p);
      for (int c = 0; c < p; ++c) M[c * kTsRows + tid] = r < end ? (double)A[r + (int64_t)c * lda] : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < p; ++j) {
      // ||x||^2 of x = M[j:, j]
      const double xr = tid >= j ? M[j * kTsRows + tid] : 0.0;
      double s2 = xr * xr;
#pragma unroll
      for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (lane == 0) red[warp] = s2;
      __syncthreads();
      double nrm2 = 0.0;
#pragma unroll
      for (int w = 0; w < kTsThreads / 32; ++w) nrm2 += red[w];
      const double alpha = M[j * kTsRows + j];
      const double nrm = sqrt(nrm2);
      __syncthreads();  // everyone has read alpha / red before they change
      if (nrm2 == 0.0) continue;
      const double beta = alpha >= 0.0 ? -nrm : nrm;
      const double v0 = alpha - beta;
      // v = x with v_j = v0; H = I - 2 v v^T / (v^T v), v^T v = nrm2 - alpha^2 + v0^2
      const double vtv = nrm2 - alpha * alpha + v0 * v0;
      const double scale = vtv > 0.0 ? 2.0 / vtv : 0.0;
      // trailing columns, one per warp at a time
      for (int c = j + 1 + warp; c < p; c += kTsThreads / 32) {
        double dot = 0.0;
        for (int r = j + lane; r < kTsRows; r += 32) {
          const double vr = r == j ? v0 : M[j * kTsRows + r];
          dot += vr * M[c * kTsRows + r];
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const double f = scale * dot;
        for (int r = j + lane; r < kTsRows; r += 32) {
          const double vr = r == j ? v0 : M[j * kTsRows + r];
          M[c * kTsRows + r] -= f * vr;
        }
      }
      __syncthreads();  // column j's reflector has been read by every warp
      if (tid == j) M[j * kTsRows + j] = beta;
      else if (tid > j) M[j * kTsRows + tid] = 0.0;
      __syncthreads();
    }
    if (end <= beg) break;
  }
  // the CTA's R: rows 0 .. p-1 of the tile (upper triangular)
  __syncthreads();
  for (int e = tid; e < p * p; e += kTsThreads) {
    const int i = e % p, j = e / p;
    double v = i <= j ? M[j * kTsRows + i] : 0.0;
    if (final_fix && M[i * kTsRows + i] < 0.0) v = -v;  // diag(R) >= 0 (kernels.py:226-230)
    Rstack[(int64_t)blockIdx.x * p + i + (int64_t)j * lds] = v;
  }
  if (final_fix && info_out && tid == 0) {
    int bad = 0;
    for (int i = 0; i < p; ++i) {
      const double d = M[i * kTsRows + i];
      if (!(fabs(d) > 0.0) || !isfinite(d)) { bad = i + 1; break; }
    }
    *info_out = bad;  // 0: R is a valid factor (replaces the Gram Cholesky's status)
  }
}

// R (p x p, ldr) <- the R factor of A (n x p); ws holds the stacked per-CTA
// factors.  cond / info as above (info may alias cond).
template <typename T>
int tsqr_r_t(int64_t n, int p, const T* A, int64_t lda, double* R, int64_t ldr, const int* cond, int* info, void* ws,
             size_t wsb, cudaStream_t st) {
  const int slab = kTsRows - p;
  int ctas = (int)std::min<int64_t>(2 * (int64_t)sm_count(), std::max<int64_t>(1, (n + slab - 1) / slab));
  const size_t need = (size_t)ctas * p * p * sizeof(double);
  RB_REQUIRE(ws && need <= wsb, "rb_tsqr_r: workspace too small");
  int64_t rows = (n + ctas - 1) / ctas;
  ctas = (int)std::max<int64_t>(1, (n + rows - 1) / rows);
  const size_t smem = ((size_t)p * kTsRows + 16) * sizeof(double);
  cudaFuncSetAttribute(tsqr_seq<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(tsqr_seq<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  double* stack = (double*)ws;
  const int64_t lds = (int64_t)ctas * p;
  RB_KLAUNCH tsqr_seq<T><<<ctas, kTsThreads, smem, st>>>(n, p, A, lda, rows, stack, lds, cond, 0, nullptr);
  RB_KLAUNCH tsqr_seq<double><<<1, kTsThreads, smem, st>>>(lds, p, stack, lds, lds, R, ldr, cond, 1, info);
  return check_launch("rb_tsqr_r");
}

int tsqr_r(int ad, int64_t n, int p, const void* A, int64_t lda, double* R, int64_t ldr, const int* cond, int* info,
           void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(n >= 1 && p >= 1 && p <= 64 && A && lda >= n && R && ldr >= p, "rb_tsqr_r: bad args (n=%lld p=%d)",
             (long long)n, p);
  return ad == RB_F32 ? tsqr_r_t<float>(n, p, (const float*)A, lda, R, ldr, cond, info, ws, wsb, st)
                      : tsqr_r_t<double>(n, p, (const double*)A, lda, R, ldr, cond, info, ws, wsb, st);
}

int potrf_upper(int p, const double* G, int64_t ldg, double* R, int64_t ldr, int* info, cudaStream_t st) {
  RB_REQUIRE(p >= 1 && p <= 128 && G && R && info && ldg >= p && ldr >= p, "rb_potrf_upper: bad args (p=%d)", p);
  const size_t smem = (size_t)p * p * sizeof(double);
  cudaFuncSetAttribute(potrf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 132 * 1024);
  RB_KLAUNCH potrf_kernel<<<1, 256, smem, st>>>(p, G, ldg, R, ldr, info);
  return check_launch("rb_potrf_upper");
}

int trsm_right(int ind, int outd, int64_t n, int p, const void* B, int64_t ldb, const double* R, int64_t ldr,
               void* X, int64_t ldx, cudaStream_t st) {
  RB_REQUIRE(n >= 0 && p >= 1 && p <= 64 && R && ldr >= p && ldb >= n && ldx >= n, "rb_trsm_right: bad args");
  if (n == 0) return RB_OK;
  if (ind == RB_F32 && outd == RB_F32) trsm_right_launch<float, float>(n, p, B, ldb, R, ldr, X, ldx, st);
  else if (ind == RB_F32) trsm_right_launch<float, double>(n, p, B, ldb, R, ldr, X, ldx, st);
  else if (outd == RB_F32) trsm_right_launch<double, float>(n, p, B, ldb, R, ldr, X, ldx, st);
  else trsm_right_launch<double, double>(n, p, B, ldb, R, ldr, X, ldx, st);
  return check_launch("rb_trsm_right");
}

int trsm_left_upper(int m, int nrhs, const double* R, int64_t ldr, double* B, int64_t ldb, int* info,
                    cudaStream_t st) {
  RB_REQUIRE(m >= 1 && nrhs >= 0 && R && B && info && ldr >= m && ldb >= m, "rb_trsm_left_upper: bad args");
  const int warps = std::max(nrhs, 1);
  RB_KLAUNCH trsm_left_upper_kernel<<<ceil_div(warps * 32, 128), 128, 0, st>>>(m, nrhs, R, ldr, B, ldb, info);
  return check_launch("rb_trsm_left_upper");
}

int geqrf_small(int m, int q, double* A, int64_t lda, double* R, int64_t ldr, void* ws, size_t wsb,
                cudaStream_t st) {
  RB_REQUIRE(q >= 1 && q <= 1024 && m >= q && A && R && lda >= m && ldr >= q, "rb_geqrf_small: bad args (m=%d q=%d)", m, q);
  RB_REQUIRE(ws && wsb >= ((size_t)m * q + q) * sizeof(double), "rb_geqrf_small: workspace");
  double* V = (double*)ws;
  RB_KLAUNCH geqrf_kernel<<<1, 1024, 0, st>>>(m, q, A, lda, R, ldr, V, V + (size_t)m * q);
  return check_launch("rb_geqrf_small");
}

int sumsq(int dt, int64_t m, int n, const void* A, int64_t lda, int minus_id, double* out, void* ws, size_t wsb,
          cudaStream_t st) {
  RB_REQUIRE(m >= 0 && n >= 0 && out && (m * n == 0 || (A && lda >= m)), "rb_sumsq: bad args");
  const int64_t tot = m * n;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>((tot + 4095) / 4096, 2 * sm_count()));
  RB_REQUIRE(ws && wsb >= (size_t)grid * sizeof(double), "rb_sumsq: workspace");
  if (dt == RB_F32) RB_KLAUNCH sumsq_partial<float><<<grid, kThreads, 0, st>>>(m, n, (const float*)A, lda, minus_id, (double*)ws);
  else RB_KLAUNCH sumsq_partial<double><<<grid, kThreads, 0, st>>>(m, n, (const double*)A, lda, minus_id, (double*)ws);
  RB_KLAUNCH sum_vec<<<1, kThreads, 0, st>>>((double*)ws, grid, out);
  return check_launch("rb_sumsq");
}

// Three binary64 sums of squares in ONE launch (the per-block finiteness
// words of P_i, S_i and R_ii, rbgs.py:380-388 via Matrix() checks): one
// CTA per matrix, column loops without integer division.
struct Mat3 {
  const double* a[3];
  int64_t lda[3];
  int64_t m[3];
  int n[3];
};

// Each CTA writes its partial into the caller's workspace; the last CTA of a
// matrix (arrival counter, also in the workspace, zeroed by the host wrapper
// in stream order) adds the partials in CTA order.  No device globals: two
// streams with their own workspaces never share state.
constexpr int kSq3Ctas = 8;

__global__ void __launch_bounds__(512) sumsq3_kernel(Mat3 M, double* __restrict__ out,
                                                     double* __restrict__ part, unsigned int* __restrict__ count) {
  // grid (3 matrices, kSq3Ctas): each CTA loops over its share of the
  // flattened m x n index with 8 independent loads in flight per thread
  // (the matrices are k x p: a column-by-column loop in one CTA was a chain
  // of dependent L2 round trips)
  __shared__ double red[16];
  __shared__ bool last;
  const int b = blockIdx.x;
  const double* __restrict__ A = M.a[b];
  const int m = (int)M.m[b];
  const int64_t lda = M.lda[b];
  const int tot = m * M.n[b];
  const int stride = gridDim.y * blockDim.x;
  double s = 0.0;
  constexpr int U = 8;
  for (int e0 = blockIdx.y * blockDim.x + threadIdx.x; e0 < tot; e0 += U * stride) {
    double v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = e0 + q * stride;
      v[q] = e < tot ? A[(int64_t)(e % m) + (int64_t)(e / m) * lda] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) s += v[q] * v[q];
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    part[b * kSq3Ctas + blockIdx.y] = s;
    __threadfence();
    last = atomicAdd(&count[b], 1u) == gridDim.y - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double t = 0.0;
    for (int q = 0; q < (int)gridDim.y; ++q) t += *(volatile double*)&part[b * kSq3Ctas + q];
    out[b] = t;
  }
}

int sumsq3(int64_t m1, int n1, const double* A1, int64_t lda1, int64_t m2, int n2, const double* A2, int64_t lda2,
           int64_t m3, int n3, const double* A3, int64_t lda3, double* out, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(out && m1 >= 0 && m2 >= 0 && m3 >= 0 && n1 >= 0 && n2 >= 0 && n3 >= 0 &&
                 (m1 * n1 == 0 || (A1 && lda1 >= m1)) && (m2 * n2 == 0 || (A2 && lda2 >= m2)) &&
                 (m3 * n3 == 0 || (A3 && lda3 >= m3)),
             "rb_sumsq3: bad args");
  constexpr size_t kPart = 3 * kSq3Ctas * sizeof(double);
  RB_REQUIRE(ws && wsb >= kPart + 4 * sizeof(unsigned int) && (uintptr_t)ws % 8 == 0, "rb_sumsq3: workspace");
  Mat3 M;
  M.a[0] = A1; M.a[1] = A2; M.a[2] = A3;
  M.lda[0] = lda1; M.lda[1] = lda2; M.lda[2] = lda3;
  M.m[0] = m1; M.m[1] = m2; M.m[2] = m3;
  M.n[0] = n1; M.n[1] = n2; M.n[2] = n3;
  RB_REQUIRE(m1 * n1 < (1ll << 31) && m2 * n2 < (1ll << 31) && m3 * n3 < (1ll << 31), "rb_sumsq3: too large");
  double* part = (double*)ws;
  unsigned int* count = (unsigned int*)((char*)ws + kPart);
  cudaMemsetAsync(count, 0, 3 * sizeof(unsigned int), st);
  RB_KLAUNCH sumsq3_kernel<<<dim3(3, kSq3Ctas), 512, 0, st>>>(M, out, part, count);
  return check_launch("rb_sumsq3");
}

int convert(int ind, int outd, int64_t m, int n, const void* X, int64_t ldx, void* Y, int64_t ldy, cudaStream_t st) {
  RB_REQUIRE(m >= 0 && n >= 0 && ldx >= m && ldy >= m, "rb_convert: bad args");
  const int64_t tot = m * n;
  if (tot == 0) return RB_OK;
  const int grid = (int)std::min<int64_t>((tot + 255) / 256, 16 * sm_count());
  if (ind == RB_F32 && outd == RB_F32) RB_KLAUNCH convert_kernel<float, float><<<grid, 256, 0, st>>>(m, n, (const float*)X, ldx, (float*)Y, ldy);
  else if (ind == RB_F32) RB_KLAUNCH convert_kernel<float, double><<<grid, 256, 0, st>>>(m, n, (const float*)X, ldx, (double*)Y, ldy);
  else if (outd == RB_F32) RB_KLAUNCH convert_kernel<double, float><<<grid, 256, 0, st>>>(m, n, (const double*)X, ldx, (float*)Y, ldy);
  else RB_KLAUNCH convert_kernel<double, double><<<grid, 256, 0, st>>>(m, n, (const double*)X, ldx, (double*)Y, ldy);
  return check_launch("rb_convert");
}

}  // namespace rb
