// K3: Step-3 projection Qp = fl(W - Q X) in the reference's elementary order
// (rbgs.py:369-370 -> kernels.py:171-209), with the two Frobenius norms of
// rbgs.py:373-374 fused in.
//
// Coarse (binary32) path: a thread owns one or two consecutive rows and all
// p column accumulators of each.  Per entry and per l the arithmetic is
//     acc = fl32(acc + fl32(q * (-x)))  ==  fl32(acc - fl32(q * x)),
// i.e. the reference's separately rounded multiply and subtract, l
// ascending, as scalar FMUL + FADD (__fmul_rn / __fadd_rn are never
// contracted).  NOTE: packed mul.rn.f32x2 + add.rn.f32x2 cannot be used for
// this -- ptxas 12.9 fuses the pair into FFMA2 even with -fmad=false (checked
// in SASS), which would break bit-identity.  The packed FFMA2 form is what
// the opt-in RB_ORDER_FMA mode uses.
// Fine (binary64) path: one row per thread, __dmul_rn / __dsub_rn.
//
// Q is streamed once (column-major, each column contiguous): per l a warp
// reads 256 contiguous bytes.  X (fp64 on entry) is rounded to the compute
// format and staged, negated, in shared memory in chunks of kLC rows.
#include "common.cuh"

namespace rb {
namespace {

constexpr int kThreads = 256;
constexpr int kLC = 32;  // X rows staged per chunk

template <typename T>
__device__ __forceinline__ float to_f32(T v) {  // binary64 -> binary32 rounds to nearest
  return static_cast<float>(v);  // double -> float rounds to nearest
}

// ---- coarse ---------------------------------------------------------------
// RPT consecutive rows per thread, PB (multiple of 4) column accumulators per
// row.  FAST = 0: reference order, acc = fl32(acc + fl32(q * (-x))) with
// __fmul_rn / __fadd_rn (FMUL + FADD, never contracted: bit-identical to
// kernels.gemm coarse).  FAST = 1: one packed FFMA2 per two columns,
// acc = fl32(acc - q x) rounded once (the survey's "FMA" variant,
// SURVEY.md section 0 finding 5; not bit-identical).
template <typename TQ, typename TW, int PB, int RPT, bool FAST>
__global__ void __launch_bounds__(kThreads)
project_coarse(int64_t n, int c, int p, const TQ* __restrict__ Q, int64_t ldq,
               const double* __restrict__ X, int64_t ldx, const TW* __restrict__ W, int64_t ldw,
               TQ* __restrict__ Qp, int64_t ldqp, double* __restrict__ partial) {
  static_assert(PB % 4 == 0, "PB multiple of 4");
  __shared__ __align__(16) float sx[kLC][PB];  // -fl32(X[l0 + l, j])
  __shared__ double red[kThreads / 32];

  const int64_t r0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * RPT;
  bool v[RPT];
#pragma unroll
  for (int r = 0; r < RPT; ++r) v[r] = r0 + r < n;

  float acc[RPT][PB];
  double w2 = 0.0;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      acc[r][j] = 0.f;
      if (j < p && v[r]) {
        const TW wv = W[r0 + r + (int64_t)j * ldw];
        w2 += (double)wv * (double)wv;
        acc[r][j] = to_f32(wv);
      }
    }

  for (int l0 = 0; l0 < c; l0 += kLC) {
    const int lc = min(kLC, c - l0);
    __syncthreads();
    for (int e = threadIdx.x; e < kLC * PB; e += kThreads) {
      const int l = e / PB, j = e % PB;
      sx[l][j] = (l < lc && j < p) ? -__double2float_rn(X[(l0 + l) + (int64_t)j * ldx]) : 0.f;
    }
    __syncthreads();
    const TQ* qcol = Q + (int64_t)l0 * ldq + r0;
#pragma unroll 2
    for (int l = 0; l < lc; ++l) {
      float q[RPT];
#pragma unroll
      for (int r = 0; r < RPT; ++r) q[r] = v[r] ? to_f32(qcol[(int64_t)l * ldq + r]) : 0.f;
      const float4* xr = reinterpret_cast<const float4*>(sx[l]);
#pragma unroll
      for (int h = 0; h < PB / 4; ++h) {
        const float4 xx = xr[h];
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          if (FAST) {
            const float2 qq = make_float2(q[r], q[r]);
            float2 a = make_float2(acc[r][4 * h], acc[r][4 * h + 1]);
            float2 b = make_float2(acc[r][4 * h + 2], acc[r][4 * h + 3]);
            a = __ffma2_rn(qq, make_float2(xx.x, xx.y), a);
            b = __ffma2_rn(qq, make_float2(xx.z, xx.w), b);
            acc[r][4 * h] = a.x;
            acc[r][4 * h + 1] = a.y;
            acc[r][4 * h + 2] = b.x;
            acc[r][4 * h + 3] = b.y;
          } else {
            acc[r][4 * h] = __fadd_rn(acc[r][4 * h], __fmul_rn(q[r], xx.x));
            acc[r][4 * h + 1] = __fadd_rn(acc[r][4 * h + 1], __fmul_rn(q[r], xx.y));
            acc[r][4 * h + 2] = __fadd_rn(acc[r][4 * h + 2], __fmul_rn(q[r], xx.z));
            acc[r][4 * h + 3] = __fadd_rn(acc[r][4 * h + 3], __fmul_rn(q[r], xx.w));
          }
        }
      }
    }
  }

  double q2 = 0.0;
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int j = 0; j < PB; ++j)
      if (j < p && v[r]) {
        Qp[r0 + r + (int64_t)j * ldqp] = (TQ)acc[r][j];
        q2 += (double)acc[r][j] * (double)acc[r][j];
      }
  if (partial) {
    const double sw = block_sum(w2, red);
    const double sq = block_sum(q2, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = sw;
      partial[2 * blockIdx.x + 1] = sq;
    }
  }
}

// ---- fine ------------------------------------------------------------------
template <typename TQ, typename TW, int PB>
__global__ void __launch_bounds__(kThreads)
project_fine(int64_t n, int c, int p, const TQ* __restrict__ Q, int64_t ldq,
             const double* __restrict__ X, int64_t ldx, const TW* __restrict__ W, int64_t ldw,
             TQ* __restrict__ Qp, int64_t ldqp, double* __restrict__ partial) {
  __shared__ double sx[kLC][PB];
  __shared__ double red[kThreads / 32];
  const int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  const bool v = r < n;
  double acc[PB];
  double w2 = 0.0;
#pragma unroll
  for (int j = 0; j < PB; ++j) {
    acc[j] = 0.0;
    if (j < p && v) {
      acc[j] = (double)W[r + j * ldw];
      w2 += acc[j] * acc[j];
    }
  }
  for (int l0 = 0; l0 < c; l0 += kLC) {
    const int lc = min(kLC, c - l0);
    __syncthreads();
    for (int e = threadIdx.x; e < kLC * PB; e += kThreads) {
      const int l = e / PB, j = e % PB;
      sx[l][j] = (l < lc && j < p) ? X[(l0 + l) + (int64_t)j * ldx] : 0.0;
    }
    __syncthreads();
    const TQ* qcol = Q + (int64_t)l0 * ldq + r;
#pragma unroll 4
    for (int l = 0; l < lc; ++l) {
      const double q = v ? (double)qcol[(int64_t)l * ldq] : 0.0;
#pragma unroll
      for (int j = 0; j < PB; ++j) acc[j] = __dsub_rn(acc[j], __dmul_rn(q, sx[l][j]));
    }
  }
  double q2 = 0.0;
#pragma unroll
  for (int j = 0; j < PB; ++j)
    if (j < p && v) {
      Qp[r + j * ldqp] = (TQ)acc[j];
      q2 += acc[j] * acc[j];
    }
  if (partial) {
    const double sw = block_sum(w2, red);
    const double sq = block_sum(q2, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = sw;
      partial[2 * blockIdx.x + 1] = sq;
    }
  }
}

// Fixed-order sum of `count` interleaved pairs into out[0..1].
__global__ void sum_pairs(const double* __restrict__ partial, int count, double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  const double sa = block_sum(a, red);
  const double sb = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = sa;
    out[1] = sb;
  }
}

template <int PB>
constexpr int rows_per_thread() { return PB <= 40 ? 2 : 1; }

template <typename TQ, typename TW, int PB>
void launch_pb(int mode, int64_t n, int c, int p, const void* Q, int64_t ldq, const double* X, int64_t ldx,
               const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* partial, cudaStream_t st) {
  if (mode == 2) {
    const int grid = ceil_div(n, kThreads);
    RB_KLAUNCH project_fine<TQ, TW, PB><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx, (const TW*)W, ldw,
                                                       (TQ*)Qp, ldqp, partial);
    return;
  }
  constexpr int RPT = rows_per_thread<PB>();
  const int grid = ceil_div(n, (int64_t)RPT * kThreads);
  if (mode == 1)
    RB_KLAUNCH project_coarse<TQ, TW, PB, RPT, true><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx,
                                                                    (const TW*)W, ldw, (TQ*)Qp, ldqp, partial);
  else
    RB_KLAUNCH project_coarse<TQ, TW, PB, RPT, false><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx,
                                                                     (const TW*)W, ldw, (TQ*)Qp, ldqp, partial);
}

template <typename TQ, typename TW>
int launch_tw(int mode, int64_t n, int c, int p, const void* Q, int64_t ldq, const double* X, int64_t ldx,
              const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* partial, cudaStream_t st) {
#define RB_PB(V)                                                                              \
  if (p <= V) {                                                                               \
    launch_pb<TQ, TW, V>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, st);       \
    return V;                                                                                 \
  }
  RB_PB(4) RB_PB(8) RB_PB(12) RB_PB(16) RB_PB(20) RB_PB(24) RB_PB(32) RB_PB(40) RB_PB(48) RB_PB(64)
#undef RB_PB
  return 0;
}

int grid_rows(int mode, int p) {
  if (mode == 2) return kThreads;
  return (p <= 40 ? 2 : 1) * kThreads;
}

}  // namespace

int project(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p, const void* Q,
            int64_t ldq, const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp,
            double* norms2, void* ws, size_t ws_bytes, cudaStream_t st) {
  RB_REQUIRE(n >= 0 && c >= 0 && p >= 1 && p <= 64, "rb_project: bad sizes n=%lld c=%d p=%d",
             (long long)n, c, p);
  RB_REQUIRE(c == 0 || (Q && ldq >= n && X && ldx >= c), "rb_project: bad Q/X");
  RB_REQUIRE(W && ldw >= n && Qp && ldqp >= n, "rb_project: bad W/Qp");
  RB_REQUIRE(order == RB_ORDER_REFERENCE || order == RB_ORDER_FMA, "rb_project: bad order %d", order);
  const int mode = compute_dtype == RB_F64 ? 2 : (order == RB_ORDER_FMA ? 1 : 0);
  const int grid = ceil_div(n, grid_rows(mode, p));
  double* partial = nullptr;
  if (norms2) {
    RB_REQUIRE(ws && ws_bytes >= (size_t)grid * 2 * sizeof(double), "rb_project: workspace");
    partial = (double*)ws;
  }
  if (n == 0) {
    if (norms2) cudaMemsetAsync(norms2, 0, 2 * sizeof(double), st);
    return check_launch("rb_project");
  }
  const bool q32 = q_dtype == RB_F32, w32 = w_dtype == RB_F32;
  if (q32 && w32) launch_tw<float, float>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, st);
  else if (q32) launch_tw<float, double>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, st);
  else if (w32) launch_tw<double, float>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, st);
  else launch_tw<double, double>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, st);
  if (norms2) RB_KLAUNCH sum_pairs<<<1, kThreads, 0, st>>>(partial, grid, norms2);
  return check_launch("rb_project");
}

}  // namespace rb
