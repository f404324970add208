// K3: Step-3 projection Qp = fl(W - Q X) in the reference's elementary order
// (rbgs.py:369-370 -> kernels.py:171-209), with the two Frobenius norms of
// rbgs.py:373-374 fused in.
//
// Coarse (binary32) path: a thread owns one or two consecutive rows and all
// p column accumulators of each.  Per entry and per l the arithmetic is
//     acc = fl32(acc + fl32(q * (-x)))  ==  fl32(acc - fl32(q * x)),
// i.e. the reference's separately rounded multiply and subtract, l
// ascending: scalar FMUL + FADD (__fmul_rn / __fadd_rn are never contracted)
// or, in the staged kernel (default), the same two roundings as packed
// FFMA2(q, -x, nz) + FADD2 with nz = -0.0f passed at run time -- ptxas
// cannot see the addend is -0 and so cannot contract the pair (it does fuse
// a literal mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 even with
// -fmad=false, checked in SASS).  RB_ORDER_REFERENCE_SCALAR forces the
// scalar form (same bits; the cross-check of the packed one).  One packed
// FFMA2 per two columns (one rounding) is the opt-in RB_ORDER_FMA mode.
// Fine (binary64) path: one row per thread, __dmul_rn / __dsub_rn.
//
// W and Qp may alias (Q' written over W_i: DeviceConfig.overwrite_w): every
// thread reads its W entries before it writes the same entries of Qp, so
// they carry no __restrict__.
//
// Q is streamed once (column-major, each column contiguous): per l a warp
// reads 256 contiguous bytes.  X (fp64 on entry) is rounded to the compute
// format and staged, negated, in shared memory in chunks of kLC rows.
#include <stdlib.h>

#include "common.cuh"
#include "tri_const.cuh"
#include "tc.cuh"

namespace rb {
namespace {

constexpr int kThreads = 256;
constexpr int kLC = 32;  // X rows staged per chunk

template <typename T>
__device__ __forceinline__ float to_f32(T v) {  // binary64 -> binary32 rounds to nearest
  return static_cast<float>(v);  // double -> float rounds to nearest
}

// ---- coarse ---------------------------------------------------------------
// RPT consecutive rows per thread, PB (multiple of 4) column accumulators
// each.  FAST = 0: reference order, acc = fl32(acc + fl32(q * (-x))) with
// __fmul_rn / __fadd_rn (FMUL + FADD, never contracted: bit-identical to
// kernels.gemm coarse).  FAST = 1: one packed FFMA2 per two columns,
// acc = fl32(acc - q x) rounded once (the survey's "FMA" variant, SURVEY.md
// section 0 finding 5; not bit-identical).
//
// The FP32 pipe is the bound (2 instructions per element step in reference
// order), so everything else is kept off the issue slots: X arrives
// pre-rounded and negated (prep_x) and is staged by cp.async, double
// buffered, in chunks of kXC rows padded with -0.0f (q = 0 there, so the
// padded steps add -0.0f: acc unchanged, signed zeros included) -- the inner
// loop has no bounds checks; Q is streamed through a two-bank register ring
// of PD rows (loads for the next PD rows in flight while the current bank
// is consumed); per l one LDS.128 broadcast feeds 8 * RPT FP instructions.
constexpr int kXC = 64;  // X rows per staged chunk

// Xs[l * PB + j] = -fl32(X[l, j]) for l < c, j < p; -0.0f elsewhere (l < cpad)
__global__ void prep_x(int c, int cpad, int p, int pb, const double* __restrict__ X, int64_t ldx,
                       float* __restrict__ Xs) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cpad * pb) return;
  const int l = e / pb, j = e % pb;
  Xs[e] = (l < c && j < p) ? -__double2float_rn(X[l + (int64_t)j * ldx]) : -0.0f;
}

// RPT >= 4: one CTA per SM with up to 255 registers; otherwise two CTAs
// per SM (<= 128 registers).  Ring depth PD rows of Q per bank.
template <typename TQ, typename TW, int PB, int RPT, bool FAST>
__global__ void __launch_bounds__(kThreads, RPT >= 4 ? 1 : 2)
project_coarse(int64_t n, int c, int p, const TQ* __restrict__ Q, int64_t ldq,
               const float* __restrict__ Xs, const TW* W, int64_t ldw,
               TQ* Qp, int64_t ldqp, double* __restrict__ partial) {
  constexpr int PD = RPT >= 2 ? 4 : 8;
  static_assert(PB % 4 == 0 && kXC % (2 * PD) == 0, "tiling");
  __shared__ __align__(16) float sx[2][kXC][PB];
  __shared__ double red[kThreads / 32];

  // rows beyond n compute on row 0 and are not stored
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
    const float4* src = reinterpret_cast<const float4*>(Xs + (int64_t)ch * kXC * PB);
    float4* dst = reinterpret_cast<float4*>(&sx[ch & 1][0][0]);
    for (int e = threadIdx.x; e < kXC * PB / 4; e += kThreads) tc::cp_async16(dst + e, src + e, 16);
    tc::cp_async_commit();
  };
  auto loadq = [&](float (&dst)[PD][RPT], int l0) {
#pragma unroll
    for (int u = 0; u < PD; ++u)
#pragma unroll
      for (int t = 0; t < RPT; ++t) dst[u][t] = l0 + u < c ? to_f32(qrow[t][(int64_t)(l0 + u) * ldq]) : 0.f;
  };
  auto step = [&](const float (&q)[PD][RPT], const float (*xs)[PB], int lim) {
#pragma unroll
    for (int u = 0; u < PD; ++u) {
      // never taken (lim >= PD), but a block boundary per row of X keeps
      // ptxas from hoisting later rows' LDS.128s into spills
      if (u >= lim) break;
      const float4* xr = reinterpret_cast<const float4*>(xs[u]);
#pragma unroll
      for (int h = 0; h < PB / 4; ++h) {
        const float4 xx = xr[h];
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          const float qq = q[u][t];
          float* a = &acc[t][4 * h];
          if (FAST) {
            const float2 q2 = make_float2(qq, qq);
            float2 lo = __ffma2_rn(q2, make_float2(xx.x, xx.y), make_float2(a[0], a[1]));
            float2 hi = __ffma2_rn(q2, make_float2(xx.z, xx.w), make_float2(a[2], a[3]));
            a[0] = lo.x;
            a[1] = lo.y;
            a[2] = hi.x;
            a[3] = hi.y;
          } else {
            a[0] = __fadd_rn(a[0], __fmul_rn(qq, xx.x));
            a[1] = __fadd_rn(a[1], __fmul_rn(qq, xx.y));
            a[2] = __fadd_rn(a[2], __fmul_rn(qq, xx.z));
            a[3] = __fadd_rn(a[3], __fmul_rn(qq, xx.w));
          }
        }
      }
    }
  };

  float qa[PD][RPT], qb[PD][RPT];
  loadq(qa, 0);
  if (nch > 0) stage(0);
  for (int ch = 0; ch < nch; ++ch) {
    tc::cp_async_wait<0>();
    __syncthreads();  // chunk ch landed for all; buffer (ch + 1) & 1 no longer read
    if (ch + 1 < nch) stage(ch + 1);
    const float(*xs)[PB] = sx[ch & 1];
    const int l0 = ch * kXC;
    const int lim = (nch - ch) * kXC;  // >= kXC
#pragma unroll 1
    for (int lb = 0; lb < kXC; lb += 2 * PD) {
      loadq(qb, l0 + lb + PD);
      step(qa, xs + lb, lim - lb);
      loadq(qa, l0 + lb + 2 * PD);
      step(qb, xs + lb + PD, lim - lb - PD);
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

// ---- coarse, staged (binary32 Q, aligned) ---------------------------------
// Same arithmetic as project_coarse, but Q never passes through registers
// ahead of use: a CTA owns R = NT / CS * RPT consecutive rows, and each stage
// (kKQ rows of X, i.e. kKQ columns of Q) arrives by bulk copies -- one per Q
// column segment (R * 4 contiguous bytes) plus the stage's pre-negated X
// rows -- completing on a per-buffer mbarrier; kQS buffers give two stages
// of look-ahead and a buffer is released by the last warp to finish it (no
// CTA barrier in the loop).  A thread owns RPT rows x PB / CS columns
// (CS column slices per row group), so per l it issues one LDS for its RPT
// q values and PB / CS / 4 LDS.128 for 2 * RPT * PB / CS FP instructions
// (RPT = 4, CS = 2 at p = 40: 6 loads per 160 FP).  The CTA covering the
// ragged end of the rows fills its stages with ordinary loads instead.
constexpr int kKQ = 12;          // l rows per stage (79 KB of stages: leaves room for a lean sketch CTA)
constexpr int kStagedRows = 512;  // rows per CTA
constexpr int kQS = 3;   // stage buffers

// Rows per CTA: the grid is cut into whole waves of resident CTAs (2 per SM
// at <= 256 threads, else 1), each CTA <= kStagedRows rows, a multiple of 4.
int staged_rows_per_cta(int64_t n, int nt) {
  const int64_t slots = (int64_t)sm_count() * (nt >= 512 ? 1 : 2);
  const int64_t waves = std::max<int64_t>(1, (n + slots * kStagedRows - 1) / (slots * kStagedRows));
  int64_t rows = (n + slots * waves - 1) / (slots * waves);
  rows = (rows + 3) / 4 * 4;
  return (int)std::min<int64_t>(std::max<int64_t>(rows, 4), kStagedRows);
}

template <int PB, int RPT, int CS, int NT>
constexpr size_t staged_smem() {
  return (size_t)kQS * (kKQ * (NT / CS) * RPT + kKQ * PB) * sizeof(float) + kQS * (sizeof(uint64_t) + 4);
}

// MODE 0: scalar FMUL + FADD; MODE 2: the same two roundings as packed
// instructions -- FFMA2(q, x, nz) with nz = -0.0f passed at run time (the
// exactly rounded product, signed zeros included: p + (-0) = p) followed by
// FADD2.  ptxas cannot see that nz is -0, so it cannot contract the pair
// into one FFMA2 (which it does for mul.rn.f32x2 + add.rn.f32x2).  Both
// packed instructions process two elements per issue slot at the scalar
// element rate, halving the FP issue pressure.  MODE 1: one FFMA2 (FMA
// order, not bit-identical).
template <typename TW, int PB, int RPT, int CS, int NT, int MODE>
__global__ void __launch_bounds__(NT, NT >= 512 ? 1 : 2)
project_staged(int64_t n, int c, int p, const float* __restrict__ Q, int64_t ldq,
               const float* __restrict__ Xs, const TW* W, int64_t ldw,
               float* Qp, int64_t ldqp, double* __restrict__ partial, float nz, float* Qf, int64_t ldqf,
               const double* __restrict__ Rf, int64_t ldrf, int pf, int rows_per_cta) {
  constexpr int PC = PB / CS;        // columns per thread
  constexpr int R = NT / CS * RPT;   // rows per CTA
  constexpr int QB = kKQ * R;        // Q floats per stage
  constexpr int XB = kKQ * PB;       // X floats per stage
  static_assert(PC % 4 == 0 && (RPT == 1 || RPT == 2 || RPT == 4) && (R * 4) % 16 == 0, "tiling");
  extern __shared__ __align__(128) float smem[];
  float* sq = smem;                                             // [kQS][kKQ][R]
  float* sx = smem + kQS * QB;                                  // [kQS][kKQ][PB]
  uint64_t* full = reinterpret_cast<uint64_t*>(sx + kQS * XB);  // [kQS]
  uint32_t* done = reinterpret_cast<uint32_t*>(full + kQS);     // [kQS] warps done
  __shared__ double red[NT / 32];

  const int cg = threadIdx.x % CS, rt = threadIdx.x / CS;
  const int jc = cg * PC;  // first column of this thread
  // Rt <= R rows per CTA (a multiple of 4 chosen by the host so the grid is
  // a whole number of waves: no partial last wave on the FP32 pipe)
  const int64_t rc = (int64_t)blockIdx.x * rows_per_cta;
  const int Rt = (int)min((int64_t)rows_per_cta, n - rc);
  const bool bulk = (Rt & 3) == 0;  // 16-byte column segments
  const int64_t rend = rc + Rt;

  if constexpr (PB <= 40) if (pf > 0) {
    // Fused Step-5 scaling of the PREVIOUS block (pf <= PB columns, the last
    // pf of Q[:, :c]): Q_(i-1) = fl32(Q'_(i-1) R^{-1}) for this CTA's rows,
    // in place, with exactly trsm_right_kernel's arithmetic (tri_solve_row:
    // binary64 registers, l ascending, R from the constant bank loaded by
    // the host wrapper).  Only this CTA reads these rows afterwards, so no
    // grid-wide ordering is needed.
    for (int rr = threadIdx.x; rr < Rt; rr += NT) {
      const int64_t row = rc + rr;
      double x[PB];
#pragma unroll
      for (int j = 0; j < PB; ++j) x[j] = j < pf ? (double)Qf[row + (int64_t)j * ldqf] : 0.0;
      tri_solve_row<PB, 1>(x, pf);  // one chain: the projection kernel is register-tight
#pragma unroll
      for (int j = 0; j < PB; ++j)
        if (j < pf) Qf[row + (int64_t)j * ldqf] = (float)x[j];
    }
    // these generic-proxy stores are read back by bulk (async-proxy) copies
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __syncthreads();
  }
  const int64_t r0 = rc + (int64_t)rt * RPT;
  bool v[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) v[t] = r0 + t < rend;

  const int nst = (c + kKQ - 1) / kKQ;
  auto issue_bulk = [&](int s) {  // one thread
    const int b = s % kQS, l0 = s * kKQ, lc = min(kKQ, c - l0);
    float* dq = sq + b * QB;
    tc::fence_proxy_async_smem();
    tc::mbar_arrive_expect_tx(&full[b], (uint32_t)((lc * Rt + XB) * sizeof(float)));
    for (int u = 0; u < lc; ++u)
      tc::bulk_g2s(dq + u * R, Q + (int64_t)(l0 + u) * ldq + rc, Rt * sizeof(float), &full[b]);
    tc::bulk_g2s(sx + b * XB, Xs + (int64_t)l0 * PB, XB * sizeof(float), &full[b]);
  };
  auto issue_tail = [&](int s) {  // all threads
    const int b = s % kQS, l0 = s * kKQ, lc = min(kKQ, c - l0);
    float* dq = sq + b * QB;
    float* dx = sx + b * XB;
    for (int e = threadIdx.x; e < lc * R; e += NT) {
      const int u = e / R, r = e % R;
      dq[e] = r < Rt ? Q[(int64_t)(l0 + u) * ldq + rc + r] : 0.f;
    }
    for (int e = threadIdx.x; e < XB; e += NT) dx[e] = Xs[(int64_t)l0 * PB + e];
  };
  if (threadIdx.x == 0) {
    for (int b = 0; b < kQS; ++b) {
      tc::mbar_init(&full[b], 1);
      done[b] = 0;
    }
    tc::mbar_fence_init();
  }
  __syncthreads();
  for (int s = 0; s < kQS && s < nst; ++s) {
    if (!bulk) issue_tail(s);
    else if (threadIdx.x == 0) issue_bulk(s);
  }
  __syncthreads();  // tail path: prologue stages written

  // W_i into the accumulators while the first stages are in flight
  float acc[RPT][PC];
  double w2 = 0.0;
#pragma unroll
  for (int t = 0; t < RPT; ++t)
#pragma unroll
    for (int j = 0; j < PC; ++j) {
      acc[t][j] = 0.f;
      if (jc + j < p && v[t]) {
        const TW wv = W[r0 + t + (int64_t)(jc + j) * ldw];
        w2 += (double)wv * (double)wv;
        acc[t][j] = to_f32(wv);
      }
    }

  for (int s = 0; s < nst; ++s) {
    const int b = s % kQS, lc = min(kKQ, c - s * kKQ);
    if (bulk) tc::mbar_wait(&full[b], (uint32_t)(s / kQS) & 1u);
    const float* qs = sq + b * QB + rt * RPT;
    const float* xs = sx + b * XB + jc;
#pragma unroll 2
    for (int u = 0; u < lc; ++u) {
      float q[RPT];
      if constexpr (RPT == 4) {
        const float4 qq = *reinterpret_cast<const float4*>(qs + u * R);
        q[0] = qq.x;
        q[1] = qq.y;
        q[2] = qq.z;
        q[3] = qq.w;
      } else if constexpr (RPT == 2) {
        const float2 qq = *reinterpret_cast<const float2*>(qs + u * R);
        q[0] = qq.x;
        q[1] = qq.y;
      } else {
        q[0] = qs[u * R];
      }
      const float4* xr = reinterpret_cast<const float4*>(xs + u * PB);
#pragma unroll
      for (int h = 0; h < PC / 4; ++h) {
        const float4 xx = xr[h];
#pragma unroll
        for (int t = 0; t < RPT; ++t) {
          float* a = &acc[t][4 * h];
          if constexpr (MODE == 1) {
            const float2 q2 = make_float2(q[t], q[t]);
            float2 lo = __ffma2_rn(q2, make_float2(xx.x, xx.y), make_float2(a[0], a[1]));
            float2 hi = __ffma2_rn(q2, make_float2(xx.z, xx.w), make_float2(a[2], a[3]));
            a[0] = lo.x;
            a[1] = lo.y;
            a[2] = hi.x;
            a[3] = hi.y;
          } else if constexpr (MODE == 2) {
            const float2 q2 = make_float2(q[t], q[t]);
            const float2 z2 = make_float2(nz, nz);
            const float2 plo = __ffma2_rn(q2, make_float2(xx.x, xx.y), z2);
            const float2 phi = __ffma2_rn(q2, make_float2(xx.z, xx.w), z2);
            const float2 lo = __fadd2_rn(make_float2(a[0], a[1]), plo);
            const float2 hi = __fadd2_rn(make_float2(a[2], a[3]), phi);
            a[0] = lo.x;
            a[1] = lo.y;
            a[2] = hi.x;
            a[3] = hi.y;
          } else {
            a[0] = __fadd_rn(a[0], __fmul_rn(q[t], xx.x));
            a[1] = __fadd_rn(a[1], __fmul_rn(q[t], xx.y));
            a[2] = __fadd_rn(a[2], __fmul_rn(q[t], xx.z));
            a[3] = __fadd_rn(a[3], __fmul_rn(q[t], xx.w));
          }
        }
      }
    }
    if (bulk) {
      // release buffer b without a CTA barrier: the last warp to finish
      // stage s refills it with stage s + kQS
      __syncwarp();
      if ((threadIdx.x & 31) == 0) {
        __threadfence_block();
        if (atomicAdd(&done[b], 1u) == NT / 32 - 1) {
          done[b] = 0;
          if (s + kQS < nst) issue_bulk(s + kQS);
        }
      }
    } else {
      __syncthreads();  // buffer b consumed by every thread
      if (s + kQS < nst) {
        issue_tail(s + kQS);
        __syncthreads();
      }
    }
  }

  double q2 = 0.0;
#pragma unroll
  for (int t = 0; t < RPT; ++t)
#pragma unroll
    for (int j = 0; j < PC; ++j)
      if (jc + j < p && v[t]) {
        Qp[r0 + t + (int64_t)(jc + j) * ldqp] = acc[t][j];
        q2 += (double)acc[t][j] * (double)acc[t][j];
      }
  if (partial) {
    const double sw = block_sum(w2, red);
    const double sq2 = block_sum(q2, red);
    if (threadIdx.x == 0) {
      partial[2 * blockIdx.x] = sw;
      partial[2 * blockIdx.x + 1] = sq2;
    }
  }
}

// ---- fine ------------------------------------------------------------------
template <typename TQ, typename TW, int PB>
__global__ void __launch_bounds__(kThreads)
project_fine(int64_t n, int c, int p, const TQ* __restrict__ Q, int64_t ldq,
             const double* __restrict__ X, int64_t ldx, const TW* W, int64_t ldw,
             TQ* Qp, int64_t ldqp, double* __restrict__ partial) {
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

// RB_PROJECT_STAGED=0 selects the register-ring kernel for binary32 Q
bool staged_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RB_PROJECT_STAGED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// RB_PROJECT_PACKED=0 selects the scalar FMUL + FADD form of the reference
// order in the staged kernel (default: packed FFMA2(-0) + FADD2, same bits)
bool packed_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RB_PROJECT_PACKED");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// rows per thread actually launched (RPT 4 is instantiated for f32/f32 only)
template <int PB>
int rpt_for(bool ff) {
  const int o = rpt_override();
  if (o == 4) return ff ? 4 : 2;
  if (o == 1 || o == 2) return o;
  return default_rpt<PB>();
}

struct FusedTrsm {
  void* Qf = nullptr;
  int64_t ldqf = 0;
  const double* Rf = nullptr;
  int64_t ldrf = 0;
  int pf = 0;
};

template <typename TQ, typename TW, int PB>
void launch_pb(int mode, int64_t n, int c, int p, const void* Q, int64_t ldq, const double* X, int64_t ldx,
               const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* partial, float* xs,
               bool staged, bool scalar, cudaStream_t st, const FusedTrsm& fz) {
  if (mode == 2) {
    const int grid = ceil_div(n, kThreads);
    RB_KLAUNCH project_fine<TQ, TW, PB><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, X, ldx, (const TW*)W,
                                                                  ldw, (TQ*)Qp, ldqp, partial);
    return;
  }
  const int cpad = ceil_div(c, kXC) * kXC;
  if (cpad > 0) RB_KLAUNCH prep_x<<<ceil_div(cpad * PB, 256), 256, 0, st>>>(c, cpad, p, PB, X, ldx, xs);
  if constexpr (sizeof(TQ) == 4) {
    if (staged) {
      // RPT x CS: rows per thread x column slices (PB / CS <= 20 columns each)
      constexpr int RPT = PB <= 20 ? 2 : 4;
      constexpr int CS = PB <= 20 ? 1 : PB <= 40 ? 2 : 4;
      constexpr int NT = kStagedRows / RPT * CS;
      // RB_PROJECT_SMEM_PAD (measurement knob): extra dynamic shared memory,
      // e.g. 120000 to force one CTA per SM
      static const size_t pad = getenv("RB_PROJECT_SMEM_PAD") ? (size_t)atol(getenv("RB_PROJECT_SMEM_PAD")) : 0;
      const size_t smem = staged_smem<PB, RPT, CS, NT>() + pad;
      const int rows = staged_rows_per_cta(n, NT);
      const int grid = ceil_div(n, (int64_t)rows);
      static bool attr = false;
      if (!attr) {
        const int mx = 227 * 1024 - 1024;  // room for the static shared arrays
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        // maximum shared-memory carveout, like the lean sketch kernel: CTAs of
        // two kernels share an SM only under one L1 / shared split
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(project_staged<TW, PB, RPT, CS, NT, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
      }
#define RB_ST(M)                                                                                  \
  RB_KLAUNCH project_staged<TW, PB, RPT, CS, NT, M><<<grid, NT, smem, st>>>(                      \
      n, c, p, (const float*)Q, ldq, xs, (const TW*)W, ldw, (float*)Qp, ldqp, partial, -0.0f,     \
      (float*)fz.Qf, fz.ldqf, fz.Rf, fz.ldrf, fz.pf, rows)
      if (mode == 1) RB_ST(1);
      else if (packed_enabled() && !scalar) RB_ST(2);
      else RB_ST(0);
#undef RB_ST
      return;
    }
  }
  const int rpt = rpt_for<PB>(sizeof(TQ) == 4 && sizeof(TW) == 4);
  const int grid = ceil_div(n, (int64_t)rpt * kThreads);
#define RB_CO(R, F)                                                                                     \
  RB_KLAUNCH project_coarse<TQ, TW, PB, R, F><<<grid, kThreads, 0, st>>>(n, c, p, (const TQ*)Q, ldq, xs, \
                                                                         (const TW*)W, ldw, (TQ*)Qp, ldqp, partial)
  if constexpr (sizeof(TQ) == 4 && sizeof(TW) == 4) {
    if (rpt == 4) {
      if (mode == 1) RB_CO(4, true); else RB_CO(4, false);
      return;
    }
  }
  if (rpt == 2) {
    if (mode == 1) RB_CO(2, true); else RB_CO(2, false);
  } else {
    if (mode == 1) RB_CO(1, true); else RB_CO(1, false);
  }
#undef RB_CO
}

template <typename TQ, typename TW>
int launch_tw(int mode, int64_t n, int c, int p, const void* Q, int64_t ldq, const double* X, int64_t ldx,
              const void* W, int64_t ldw, void* Qp, int64_t ldqp, double* partial, float* xs, bool staged,
              bool scalar, cudaStream_t st, const FusedTrsm& fz = FusedTrsm()) {
#define RB_PB(V)                                                                                    \
  if (p <= V) {                                                                                     \
    launch_pb<TQ, TW, V>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, xs, staged, scalar, st, fz); \
    return V;                                                                                       \
  }
  RB_PB(4) RB_PB(8) RB_PB(12) RB_PB(16) RB_PB(20) RB_PB(24) RB_PB(32) RB_PB(40) RB_PB(48) RB_PB(64)
#undef RB_PB
  return 0;
}

template <int PB>
int rows_for(bool ff) { return rpt_for<PB>(ff) * kThreads; }

int grid_rows(int mode, int p, bool ff) {
  if (mode == 2) return kThreads;
  if (p <= 4) return rows_for<4>(ff);
  if (p <= 8) return rows_for<8>(ff);
  if (p <= 12) return rows_for<12>(ff);
  if (p <= 16) return rows_for<16>(ff);
  if (p <= 20) return rows_for<20>(ff);
  if (p <= 24) return rows_for<24>(ff);
  if (p <= 32) return rows_for<32>(ff);
  if (p <= 40) return rows_for<40>(ff);
  if (p <= 48) return rows_for<48>(ff);
  return rows_for<64>(ff);
}

}  // namespace

int trsm_right(int, int, int64_t, int, const void*, int64_t, const double*, int64_t, void*, int64_t, cudaStream_t);
int project_tc_launch(int w_dtype, int64_t n, int c, int p, const float* Q, int64_t ldq, const double* X,
                      int64_t ldx, const void* W, int64_t ldw, float* Qp, int64_t ldqp, double* norms2, void* ws,
                      size_t wsb, cudaStream_t st, double* partial_out, int* grid_out);
size_t project_tc_ws_bytes(int c, int p);

namespace {
// norms2 = (sum of the tensor-core kernel's CTA pairs) + (the tail call's pair)
__global__ void sum_pairs_plus(const double* __restrict__ partial, int count, const double* __restrict__ extra,
                               double* __restrict__ out) {
  __shared__ double red[kThreads / 32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    a += partial[2 * i];
    b += partial[2 * i + 1];
  }
  const double sa = block_sum(a, red);
  const double sb = block_sum(b, red);
  if (threadIdx.x == 0) {
    out[0] = sa + (extra ? extra[0] : 0.0);
    out[1] = sb + (extra ? extra[1] : 0.0);
  }
}

int project_impl(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p, const void* Q,
                 int64_t ldq, const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp,
                 double* norms2, void* ws, size_t ws_bytes, cudaStream_t st, const FusedTrsm& fz);
}  // namespace

int project(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p, const void* Q,
            int64_t ldq, const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp,
            double* norms2, void* ws, size_t ws_bytes, cudaStream_t st) {
  return project_impl(q_dtype, w_dtype, compute_dtype, order, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, norms2,
                      ws, ws_bytes, st, FusedTrsm());
}

// Step 3 of block i with the Step-5 scaling of block i-1 fused in front:
// Qf (the last pf columns of Q[:, :c], i.e. Q'_(i-1) in place) becomes
// fl32(Q'_(i-1) Rf^{-1}) row by row inside the staged projection's CTAs, so
// the scaled block is written and re-read while L2-hot and its DFMA /
// shared-load work overlaps the other resident CTA's FP32 work.  Bitwise
// the same as rb_trsm_right followed by rb_project.  Falls back to exactly
// that pair when the staged kernel does not apply.
int project_trsm(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p, const void* Q,
                 int64_t ldq, const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp,
                 double* norms2, void* Qf, int64_t ldqf, const double* Rf, int64_t ldrf, int pf, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
  RB_REQUIRE(pf >= 1 && pf <= 64 && pf <= c && Qf && Rf && ldrf >= pf && ldqf >= n,
             "rb_project_trsm: bad previous block (pf=%d c=%d)", pf, c);
  const bool aligned = (uintptr_t)Q % 16 == 0 && ldq % 4 == 0;
  const bool fusable = q_dtype == RB_F32 && compute_dtype == RB_F32 && aligned && rpt_override() == 0 &&
                       staged_enabled() && p <= 40 && pf <= p && ldqf == ldq &&
                       (const char*)Qf == (const char*)Q + (size_t)(c - pf) * ldq * sizeof(float);
  if (!fusable) {
    const int rc = trsm_right(q_dtype, q_dtype, n, pf, Qf, ldqf, Rf, ldrf, Qf, ldqf, st);
    if (rc != RB_OK) return rc;
    return project(q_dtype, w_dtype, compute_dtype, order, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, norms2, ws,
                   ws_bytes, st);
  }
  std::lock_guard<std::mutex> lock(tri_mutex());
  const int lrc = load_tri_const_locked(pf, Rf, ldrf, st);
  if (lrc != RB_OK) return lrc;
  FusedTrsm fz;
  fz.Qf = Qf;
  fz.ldqf = ldqf;
  fz.Rf = Rf;
  fz.ldrf = ldrf;
  fz.pf = pf;
  const int rc = project_impl(q_dtype, w_dtype, compute_dtype, order, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp,
                              norms2, ws, ws_bytes, st, fz);
  tri_const_done_locked(st);
  return rc;
}

namespace {
int project_impl(int q_dtype, int w_dtype, int compute_dtype, int order, int64_t n, int c, int p, const void* Q,
                 int64_t ldq, const double* X, int64_t ldx, const void* W, int64_t ldw, void* Qp, int64_t ldqp,
                 double* norms2, void* ws, size_t ws_bytes, cudaStream_t st, const FusedTrsm& fz) {
  RB_REQUIRE(n >= 0 && c >= 0 && p >= 1 && p <= 64, "rb_project: bad sizes n=%lld c=%d p=%d",
             (long long)n, c, p);
  RB_REQUIRE(c == 0 || (Q && ldq >= n && X && ldx >= c), "rb_project: bad Q/X");
  RB_REQUIRE(W && ldw >= n && Qp && ldqp >= n, "rb_project: bad W/Qp");
  RB_REQUIRE(order == RB_ORDER_REFERENCE || order == RB_ORDER_FMA || order == RB_ORDER_REFERENCE_SCALAR ||
                 order == RB_ORDER_TC,
             "rb_project: bad order %d", order);
  if (order == RB_ORDER_TC) {
    // tensor pipe, 3xTF32 (project_tc.cu): binary32 Q with 16-B aligned
    // columns; rows past the last whole 128-row tile and every other
    // layout take the FMA order on the CUDA cores
    const bool ok = compute_dtype == RB_F32 && q_dtype == RB_F32 && c > 0 && (uintptr_t)Q % 16 == 0 &&
                    ldq % 4 == 0 && fz.pf == 0 && n >= 128;
    if (!ok)
      return project_impl(q_dtype, w_dtype, compute_dtype, RB_ORDER_FMA, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp,
                          norms2, ws, ws_bytes, st, fz);
    const int64_t nt = n / 128 * 128;
    const size_t tcb = (project_tc_ws_bytes(c, p) + 255) / 256 * 256;
    RB_REQUIRE(ws && ws_bytes >= tcb + 256 && (uintptr_t)ws % 256 == 0, "rb_project (tc): workspace too small");
    int grid = 0;
    int rc = project_tc_launch(w_dtype, nt, c, p, (const float*)Q, ldq, X, ldx, W, ldw, (float*)Qp, ldqp, norms2, ws,
                               tcb, st, nullptr, &grid);
    if (rc != RB_OK) return rc;
    double* tailn = norms2 ? (double*)((char*)ws + tcb) : nullptr;  // 2 doubles
    if (nt < n) {
      const size_t esw = w_dtype == RB_F32 ? 4 : 8;
      rc = project_impl(q_dtype, w_dtype, compute_dtype, RB_ORDER_FMA, n - nt, c, p, (const float*)Q + nt, ldq, X,
                        ldx, (const char*)W + nt * esw, ldw, (float*)Qp + nt, ldqp, tailn,
                        (char*)ws + tcb + 256, ws_bytes - tcb - 256, st, fz);
      if (rc != RB_OK) return rc;
    } else if (tailn) {
      cudaMemsetAsync(tailn, 0, 2 * sizeof(double), st);
    }
    if (norms2) RB_KLAUNCH sum_pairs_plus<<<1, kThreads, 0, st>>>((const double*)ws, grid, tailn, norms2);
    return check_launch("rb_project (tc)");
  }
  const int mode = compute_dtype == RB_F64 ? 2 : (order == RB_ORDER_FMA ? 1 : 0);
  const bool scalar = order == RB_ORDER_REFERENCE_SCALAR;
  const bool q32 = q_dtype == RB_F32, w32 = w_dtype == RB_F32;
  // binary32 Q with 16-B aligned columns streams through the staged kernel
  const bool staged = mode != 2 && q32 && c > 0 && rpt_override() == 0 && (uintptr_t)Q % 16 == 0 &&
                      ldq % 4 == 0 && staged_enabled();
  const int grid = staged ? ceil_div(n, (int64_t)staged_rows_per_cta(n, p > 40 ? 512 : 256))
                          : ceil_div(n, grid_rows(mode, p, q32 && w32));
  // workspace: [per-CTA norm pairs | staged -fl32(X), cpad x 64 floats]
  const size_t part_bytes = norms2 ? ((size_t)grid * 2 * sizeof(double) + 255) / 256 * 256 : 0;
  const size_t xs_bytes = mode == 2 ? 0 : (size_t)ceil_div(c, kXC) * kXC * 64 * sizeof(float);
  RB_REQUIRE(part_bytes + xs_bytes == 0 || (ws && ws_bytes >= part_bytes + xs_bytes && (uintptr_t)ws % 16 == 0),
             "rb_project: workspace too small (%zu < %zu)", ws_bytes, part_bytes + xs_bytes);
  double* partial = norms2 ? (double*)ws : nullptr;
  float* xs = xs_bytes ? (float*)((char*)ws + part_bytes) : nullptr;
  if (n == 0) {
    if (norms2) cudaMemsetAsync(norms2, 0, 2 * sizeof(double), st);
    return check_launch("rb_project");
  }
  RB_REQUIRE(fz.pf == 0 || staged, "rb_project: fused scaling needs the staged kernel");
  if (q32 && w32) launch_tw<float, float>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, xs, staged, scalar, st, fz);
  else if (q32) launch_tw<float, double>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, xs, staged, scalar, st, fz);
  else if (w32) launch_tw<double, float>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, xs, staged, scalar, st);
  else launch_tw<double, double>(mode, n, c, p, Q, ldq, X, ldx, W, ldw, Qp, ldqp, partial, xs, staged, scalar, st);
  if (norms2) RB_KLAUNCH sum_pairs<<<1, kThreads, 0, st>>>(partial, grid, norms2);
  return check_launch("rb_project");
}
}  // namespace

}  // namespace rb
