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
#include <stdlib.h>

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
// One row per thread, PB (multiple of 4) column accumulators.  FAST = 0:
// reference order, acc = fl32(acc + fl32(q * (-x))) with __fmul_rn /
// __fadd_rn (FMUL + FADD, never contracted: bit-identical to kernels.gemm
// coarse).  FAST = 1: one packed FFMA2 per two columns, acc = fl32(acc - q x)
// rounded once (the survey's "FMA" variant, SURVEY.md section 0 finding 5;
// not bit-identical).  Q is streamed with a kPD-deep register prefetch ring
// that runs across the X-chunk boundaries; X chunks are double-buffered.
constexpr int kXC = 64;  // X rows per staged chunk
constexpr int kPD = 8;   // Q prefetch depth (loads in flight per thread)

template <typename TQ, typename TW, int PB, int RPT, bool FAST>
__global__ void __launch_bounds__(kThreads, 2)
project_coarse(int64_t n, int c, int p, const TQ* __restrict__ Q, int64_t ldq,
               const double* __restrict__ X, int64_t ldx, const TW* __restrict__ W, int64_t ldw,
               TQ* __restrict__ Qp, int64_t ldqp, double* __restrict__ partial) {
  static_assert(PB % 4 == 0, "PB multiple of 4");
  __shared__ __align__(16) float sx[2][kXC][PB];  // -fl32(X[l, j]), double-buffered
  __shared__ double red[kThreads / 32];

  // RPT consecutive rows per thread (each x broadcast from shared memory
  // feeds RPT rows); rows beyond n compute on row 0 and are not stored
  const int64_t r0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * RPT;
  bool v[RPT];
  const TQ* qrow[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    v[t] = r0 + t < n;
    qrow[t] = Q + (v[t] ? r0 + t : 0);
  }

  float acc[RPT][PB];
  double w2 = 0.0;
#pragma unroll
  for (int t = 0; t < RPT; ++t)
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      acc[t][j] = 0.f;
      if (j < p && v[t]) {
        const TW wv = W[r0 + t + (int64_t)j * ldw];
        w2 += (double)wv * (double)wv;
        acc[t][j] = to_f32(wv);
      }
    }

  const int nch = (c + kXC - 1) / kXC;
  auto stage = [&](int ch) {
    const int l0 = ch * kXC, lc = min(kXC, c - l0);
    float(*dst)[PB] = sx[ch & 1];
    for (int e = threadIdx.x; e < kXC * PB; e += kThreads) {
      const int l = e / PB, j = e % PB;
      dst[l][j] = (l < lc && j < p) ? -__double2float_rn(X[(l0 + l) + (int64_t)j * ldx]) : 0.f;
    }
  };
  float qbuf[kPD][RPT];
#pragma unroll
  for (int u = 0; u < kPD; ++u)
#pragma unroll
    for (int t = 0; t < RPT; ++t) qbuf[u][t] = u < c ? to_f32(qrow[t][(int64_t)u * ldq]) : 0.f;
  if (nch > 0) stage(0);
  for (int ch = 0; ch < nch; ++ch) {
    __syncthreads();  // chunk ch staged; buffer (ch + 1) & 1 no longer read
    if (ch + 1 < nch) stage(ch + 1);
    const int l0 = ch * kXC, lc = min(kXC, c - l0);
    const float(*xs)[PB] = sx[ch & 1];
    for (int lb = 0; lb < lc; lb += kPD) {
      float qc[kPD][RPT];
#pragma unroll
      for (int u = 0; u < kPD; ++u)
#pragma unroll
        for (int t = 0; t < RPT; ++t) qc[u][t] = qbuf[u][t];
#pragma unroll
      for (int u = 0; u < kPD; ++u) {
        const int ln = l0 + lb + kPD + u;
#pragma unroll
        for (int t = 0; t < RPT; ++t) qbuf[u][t] = ln < c ? to_f32(qrow[t][(int64_t)ln * ldq]) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < kPD; ++u) {
        if (lb + u < lc) {
          const float4* xr = reinterpret_cast<const float4*>(xs[lb + u]);
#pragma unroll
          for (int h = 0; h < PB / 4; ++h) {
            const float4 xx = xr[h];
#pragma unroll
            for (int t = 0; t < RPT; ++t) {
              const float q = qc[u][t];
              float* a = &acc[t][4 * h];
              if (FAST) {
                const float2 qq = make_float2(q, q);
                float2 lo = __ffma2_rn(qq, make_float2(xx.x, xx.y), make_float2(a[0], a[1]));
                float2 hi = __ffma2_rn(qq, make_float2(xx.z, xx.w), make_float2(a[2], a[3]));
                a[0] = lo.x;
                a[1] = lo.y;
                a[2] = hi.x;
                a[3] = hi.y;
              } else {
                a[0] = __fadd_rn(a[0], __fmul_rn(q, xx.x));
                a[1] = __fadd_rn(a[1], __fmul_rn(q, xx.y));
                a[2] = __fadd_rn(a[2], __fmul_rn(q, xx.z));
                a[3] = __fadd_rn(a[3], __fmul_rn(q, xx.w));
              }
            }
          }
        }
      }
    }
  }

  double q2 = 0.0;
#pragma unroll
  for (int t = 0; t < RPT; ++t)
#pragma unroll
    for (int j = 0; j < PB; ++j)
      if (j < p && v[t]) {
        Qp[r0 + t + (int64_t)j * ldqp] = (TQ)acc[t][j];
        q2 += (double)acc[t][j] * (double)acc[t][j];
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

// rows per thread for the coarse kernel: two for narrow blocks (halves the
// shared-memory broadcasts per FP instruction), one when the accumulators
// would not fit two CTAs per SM.  Selectable at runtime via RB_PROJECT_RPT
// for measurement.
template <int PB>
constexpr int default_rpt() { return PB <= 40 ? 2 : 1; }

int rpt_override() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("RB_PROJECT_RPT");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <typename TQ, typename TW, int PB>
void launch_pb(int mode, int64_t n, int c, int p, const void* Q, int64_t ldq, const double* X, int64_t ldx,
               const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* partial, cudaStream_t st) {
  if (mode == 2) {
    const int grid = ceil_div(n, kThreads);
    RB_KLAUNCH project_fine<TQ, TW, PB><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx, (const TW*)W,
                                                                  ldw, (TQ*)Qp, ldqp, partial);
    return;
  }
  const int rpt = rpt_override() > 0 ? rpt_override() : default_rpt<PB>();
  const int grid = ceil_div(n, (int64_t)rpt * kThreads);
#define RB_CO(R, F)                                                                                    \
  RB_KLAUNCH project_coarse<TQ, TW, PB, R, F><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx, \
                                                                         (const TW*)W, ldw, (TQ*)Qp, ldqp, partial)
  if (rpt == 2) {
    if (mode == 1) RB_CO(2, true); else RB_CO(2, false);
  } else {
    if (mode == 1) RB_CO(1, true); else RB_CO(1, false);
  }
#undef RB_CO
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

template <int PB>
int rows_for() { return (rpt_override() > 0 ? rpt_override() : default_rpt<PB>()) * kThreads; }

int grid_rows(int mode, int p) {
  if (mode == 2) return kThreads;
  if (p <= 4) return rows_for<4>();
  if (p <= 8) return rows_for<8>();
  if (p <= 12) return rows_for<12>();
  if (p <= 16) return rows_for<16>();
  if (p <= 20) return rows_for<20>();
  if (p <= 24) return rows_for<24>();
  if (p <= 32) return rows_for<32>();
  if (p <= 40) return rows_for<40>();
  if (p <= 48) return rows_for<48>();
  return rows_for<64>();
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
