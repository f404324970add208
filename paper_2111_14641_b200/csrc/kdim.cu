// The k-dimensional steps of a block, hand-written for sm_100a (no library
// GEMMs on the per-block path):
//
//   rb_ls_richardson        Step 2, l sweeps X <- X + S^T (P - S X) from
//                           X = 0 (rbgs.py:144-156) as ONE cooperative
//                           launch: every GEMM is split over the K
//                           dimension across the whole grid, partial tiles
//                           go to the caller's workspace and are summed in
//                           split order (deterministic), grid barriers
//                           separate the phases.
//   rb_sketched_cholqr_small  one sketched-CholQR pass on the k x p sketch
//                           (rbgs.py:282-289): G = S'^T S' (split-K over the
//                           grid), R = chol(G) with dpotrf semantics
//                           (kernels.py:234-247; info = first bad column),
//                           Sout = S' R^{-1} -- ONE cooperative launch.
//   rb_certify              Step 7 (rbgs.py:428-443): ||I - S^T S||_F^2,
//                           ||P - S R||_F^2, ||P||_F^2 -- ONE cooperative
//                           launch.
//
// Arithmetic: binary64 DFMA on the CUDA cores (B200's FP64 tensor rate is
// the same as its DFMA rate, and these shapes -- p <= 64 columns, K <= a
// few thousand -- are latency-, not throughput-bound).  Every reduction has
// a fixed order, so results are bit-reproducible run to run.  The numpy
// expression order is kept where it rounds: T = P - (S X) (the product is
// formed, then subtracted), X = X + (S^T T).
#include <cooperative_groups.h>

#include <type_traits>

#include "common.cuh"

namespace cg = cooperative_groups;

// RB_KDIM_TRACE (tools/kdim_trace.cu only): CTA 0 records %globaltimer at
// phase boundaries into g_kdim_trace.
#ifdef RB_KDIM_TRACE
__device__ unsigned long long g_kdim_trace[256];
__device__ __forceinline__ void kdim_mark(int slot) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_kdim_trace[slot & 255] = t;
  }
}
#define KDIM_MARK(s) kdim_mark(s)
#else
#define KDIM_MARK(s) ((void)0)
#endif

namespace rb {

int sm_count();
int cross(int ad, int bd, int64_t n, int p, int q, const void* A, int64_t lda, const void* B, int64_t ldb,
          double* out, int64_t ldo, int acc, void* ws, size_t wsb, cudaStream_t st);

namespace {

constexpr int kKT = 256;  // threads per CTA
constexpr int kKC = 32;   // K rows staged per chunk
constexpr int kTM = 64;   // output rows per tile

// One TM x PB output tile of op(A) B over the K range [kb, ke):
//   TRANS_A = false: op(A)[i, kk] = A[i + kk * lda]   (A is M x K)
//   TRANS_A = true : op(A)[i, kk] = A[kk + i * lda]   (A is K x M, op = ^T)
//   B[kk, j] = B[kk + j * ldb]                        (K x N)
// Thread t owns rows 2 (t / 8) + {0, 1} and columns t % 8 + 8 ci, ci < PB / 8,
// accumulated in ascending kk within the range.  Rows >= mrows / columns
// >= ncols are computed on zeros.
template <int PB, bool TRANS_A>
__device__ __forceinline__ void tile_gemm(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                                          int64_t ldb, int m0, int mrows, int ncols, int64_t kb, int64_t ke,
                                          double (&acc)[2][PB / 8], double* smem) {
  double* sA = smem;             // [kKC][kTM]
  double* sB = smem + kKC * kTM; // [kKC][PB]
  const int tid = threadIdx.x;
  const int ty = tid >> 3, tx = tid & 7;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < PB / 8; ++b) acc[a][b] = 0.0;
  for (int64_t k0 = kb; k0 < ke; k0 += kKC) {
    const int kc = (int)min((int64_t)kKC, ke - k0);
    __syncthreads();
    for (int e = tid; e < kKC * kTM; e += kKT) {
      int i, kk;
      if (TRANS_A) { kk = e % kKC; i = e / kKC; } else { i = e % kTM; kk = e / kTM; }
      double v = 0.0;
      if (i < mrows && kk < kc) v = TRANS_A ? A[(k0 + kk) + (int64_t)(m0 + i) * lda] : A[(m0 + i) + (k0 + kk) * lda];
      sA[kk * kTM + i] = v;
    }
    for (int e = tid; e < kKC * PB; e += kKT) {
      const int kk = e % kKC, j = e / kKC;
      sB[kk * PB + j] = (j < ncols && kk < kc) ? B[(k0 + kk) + (int64_t)j * ldb] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < kKC; ++kk) {
      const double a0 = sA[kk * kTM + 2 * ty], a1 = sA[kk * kTM + 2 * ty + 1];
#pragma unroll
      for (int ci = 0; ci < PB / 8; ++ci) {
        const double b = sB[kk * PB + tx + 8 * ci];
        acc[0][ci] = fma(a0, b, acc[0][ci]);
        acc[1][ci] = fma(a1, b, acc[1][ci]);
      }
    }
  }
}

template <int PB>
constexpr size_t tile_smem() { return (size_t)kKC * (kTM + PB) * sizeof(double); }

// K ranges: `splits` contiguous ranges of a multiple of kKC rows each.
__device__ __forceinline__ void split_range(int64_t K, int splits, int s, int64_t& kb, int64_t& ke) {
  const int64_t chunks = (K + kKC - 1) / kKC;
  const int64_t per = (chunks + splits - 1) / splits;
  kb = min(K, (int64_t)s * per * kKC);
  ke = min(K, (int64_t)(s + 1) * per * kKC);
}

// Store a tile's partial: ws_tile[j * kTM + i] (column-major kTM x PB).
template <int PB>
__device__ __forceinline__ void store_partial(double* __restrict__ dst, const double (&acc)[2][PB / 8]) {
  const int ty = threadIdx.x >> 3, tx = threadIdx.x & 7;
#pragma unroll
  for (int ci = 0; ci < PB / 8; ++ci) {
    dst[(tx + 8 * ci) * kTM + 2 * ty] = acc[0][ci];
    dst[(tx + 8 * ci) * kTM + 2 * ty + 1] = acc[1][ci];
  }
}

// Sum of the splits of element (i, j) of tile `t` in split order.
template <int PB>
__device__ __forceinline__ double sum_splits(const double* __restrict__ ws, int tiles, int splits, int t, int i,
                                             int j) {
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += ws[((int64_t)q * tiles + t) * (kTM * PB) + j * kTM + i];
  return s;
}

// Split counts: enough (tile, split) items to cover the grid, each split at
// least kKC rows.
__device__ __forceinline__ int splits_for(int tiles, int64_t K, int grid) {
  const int64_t chunks = max((int64_t)1, (K + kKC - 1) / kKC);
  return (int)max((int64_t)1, min(chunks, (int64_t)((grid + tiles - 1) / tiles)));
}

// ============================ full-K tile items ==============================
// An item computes one MR x PB output tile of op(A) B over the WHOLE K range
// inside one CTA -- no split over CTAs, hence no cross-CTA partial
// reductions (their chains of dependent L2 round trips dominated the split-K
// versions of these small GEMMs).  The CTA's 256 threads form KG K-groups of
// TG = 256 / KG threads; a K-group thread owns 2 rows x PB / 8 columns and
// the chunk's kk in its slice; chunks of kIC rows stream through two
// shared-memory stages by 8-byte cp.async (the next chunk in flight while
// the current one is multiplied).  The K-groups' tiles are added in group
// order through shared memory: every output is a fixed-order sum.
//   TN = false: op(A)[i, kk] = A[i + kk * lda]  (rows of S: T = P - S X)
//   TN = true : op(A)[i, kk] = A[kk + i * lda]  (columns of S: S^T T, S^T S)
constexpr int kIC = 128;  // K rows per chunk
constexpr int kIP = kIC + 2;  // padded K stride (16-B aligned rows, conflict-free column reads)

template <int PB, int MR>
struct ItemSmem {
  static constexpr int KG = 256 / (MR / 2 * 8);
  double a[2][MR * kIP];      // NN: [kk][i] (stride MR), TN: [i][kk] (stride kIP)
  double b[2][PB * kIP];      // [j][kk]
  double red[KG][MR * PB];
};

__device__ __forceinline__ void cpa8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Result: sm.red[0][j * MR + i] (valid rows / columns only), ready after the
// function returns (ends with a barrier).
template <int PB, int MR, bool TN>
__device__ void tile_item(const double* __restrict__ A, int64_t lda, const double* __restrict__ B, int64_t ldb,
                          int m0, int mrows, int ncols, int64_t K, ItemSmem<PB, MR>& sm) {
  constexpr int KG = ItemSmem<PB, MR>::KG, TG = 256 / KG, SL = kIC / KG;
  const int tid = threadIdx.x, g = tid / TG, u = tid % TG;
  const int rg = u % (MR / 2), cg = u / (MR / 2);  // rows 2 rg, 2 rg + 1; columns cg + 8 ci
  double acc[2][PB / 8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < PB / 8; ++b) acc[a][b] = 0.0;
  const int nch = (int)((K + kIC - 1) / kIC);
  auto issue = [&](int ch) {
    const int st = ch & 1;
    const int64_t k0 = (int64_t)ch * kIC;
    const int kc = (int)min((int64_t)kIC, K - k0);
    double* sa = sm.a[st];
    double* sb = sm.b[st];
    for (int e = tid; e < MR * kIC; e += 256) {
      int i, kk;
      if (TN) { kk = e % kIC; i = e / kIC; } else { i = e % MR; kk = e / MR; }
      double* dst = TN ? &sa[i * kIP + kk] : &sa[kk * MR + i];
      if (i < mrows && kk < kc) cpa8(dst, TN ? &A[(k0 + kk) + (int64_t)(m0 + i) * lda] : &A[(m0 + i) + (k0 + kk) * lda]);
      else *dst = 0.0;
    }
    for (int e = tid; e < PB * kIC; e += 256) {
      const int kk = e % kIC, j = e / kIC;
      if (j < ncols && kk < kc) cpa8(&sb[j * kIP + kk], &B[(k0 + kk) + (int64_t)j * ldb]);
      else sb[j * kIP + kk] = 0.0;
    }
    cpa_commit();
  };
  if (nch > 0) issue(0);
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      issue(ch + 1);
      cpa_wait<1>();
    } else {
      cpa_wait<0>();
    }
    __syncthreads();
    const double* sa = sm.a[ch & 1];
    const double* sb = sm.b[ch & 1];
#pragma unroll 4
    for (int q = 0; q < SL; ++q) {
      const int kk = g * SL + q;
      double a0, a1;
      if (TN) {
        a0 = sa[(2 * rg) * kIP + kk];
        a1 = sa[(2 * rg + 1) * kIP + kk];
      } else {
        const double2 aa = *reinterpret_cast<const double2*>(&sa[kk * MR + 2 * rg]);
        a0 = aa.x;
        a1 = aa.y;
      }
#pragma unroll
      for (int ci = 0; ci < PB / 8; ++ci) {
        const double b = sb[(cg + 8 * ci) * kIP + kk];
        acc[0][ci] = fma(a0, b, acc[0][ci]);
        acc[1][ci] = fma(a1, b, acc[1][ci]);
      }
    }
    __syncthreads();  // stage (ch & 1) is reissued two chunks later
  }
#pragma unroll
  for (int ci = 0; ci < PB / 8; ++ci) {
    sm.red[g][(cg + 8 * ci) * MR + 2 * rg] = acc[0][ci];
    sm.red[g][(cg + 8 * ci) * MR + 2 * rg + 1] = acc[1][ci];
  }
  __syncthreads();
  for (int e = tid; e < MR * PB; e += 256) {
    double s = sm.red[0][e];
#pragma unroll
    for (int q = 1; q < KG; ++q) s += sm.red[q][e];
    sm.red[0][e] = s;
  }
  __syncthreads();
}

// ============================ Richardson ====================================
// Per sweep two phases, each one item per CTA (grid-stride if there are
// more), separated by grid barriers:
//   T = P - (S X)      items: 16-row tiles of T, K = c
//   X = X + (S^T T)    items:  8-row tiles of X, K = k
template <int PB>
struct RichSmem {
  union {
    ItemSmem<PB, 16> nn;
    ItemSmem<PB, 8> tn;
  };
};

template <int PB>
__global__ void __launch_bounds__(256, 1)
richardson_v3(int k, int c, int p, const double* __restrict__ S, int64_t lds, const double* __restrict__ P,
              int64_t ldp, int l, double* __restrict__ X, int64_t ldx, double* __restrict__ T, int64_t ldt) {
  extern __shared__ __align__(16) unsigned char smraw[];
  RichSmem<PB>& sm = *reinterpret_cast<RichSmem<PB>*>(smraw);
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int tilesT = (k + 15) / 16, tilesX = (c + 7) / 8;
  for (int sweep = 0; sweep < l; ++sweep) {
    if (sweep > 0) {
      for (int t = blockIdx.x; t < tilesT; t += G) {
        const int mrows = min(16, k - 16 * t);
        tile_item<PB, 16, false>(S + 16 * t, lds, X, ldx, 0, mrows, p, c, sm.nn);
        for (int e = threadIdx.x; e < mrows * p; e += 256) {
          const int i = e % mrows, j = e / mrows;
          const int64_t r = 16 * t + i;
          T[r + (int64_t)j * ldt] = P[r + (int64_t)j * ldp] - sm.nn.red[0][j * 16 + i];
        }
        __syncthreads();
      }
      grid.sync();
    }
    // sweep 0: X = S^T P (X = 0 and P - S 0 = P exactly)
    const double* Tin = sweep == 0 ? P : T;
    const int64_t ldtin = sweep == 0 ? ldp : ldt;
    for (int t = blockIdx.x; t < tilesX; t += G) {
      const int mrows = min(8, c - 8 * t);
      tile_item<PB, 8, true>(S + (int64_t)8 * t * lds, lds, Tin, ldtin, 0, mrows, p, k, sm.tn);
      for (int e = threadIdx.x; e < mrows * p; e += 256) {
        const int i = e % mrows, j = e / mrows;
        double* xp = X + (8 * t + i) + (int64_t)j * ldx;
        const double v = sm.tn.red[0][j * 8 + i];
        *xp = sweep == 0 ? v : *xp + v;
      }
      __syncthreads();
    }
    if (sweep + 1 < l) grid.sync();
  }
}

// ---- Richardson, v4: S resident in shared memory ------------------------------
// S (k x c) is cut into an R x C grid of blocks, one per CTA (R C <= grid),
// loaded ONCE into that CTA's shared memory and kept there for all l
// sweeps; per sweep only the small operands move (X c x p, T k x p, both
// L2-resident):
//   A  CTA (r, cb): partial T_r^(cb) = S_(r,cb) X_cb   -> ws   | barrier
//      every CTA: T = P - sum_cb (cb ascending), grid-stride  | barrier
//   B  CTA (r, cb): partial X_cb^(r) = S_(r,cb)^T T_r  -> ws   | barrier
//      every CTA: X = X + sum_r (r ascending), grid-stride    | barrier
// Fixed summation orders throughout (deterministic).  In-block products:
// a thread owns up to 8 rows x 4 consecutive columns of the block's output.
constexpr int kV4Smem = 200 * 1024;
constexpr int kV4T = 256;  // threads per CTA of richardson_v4 (DMMA saturates with few warps)

struct V4Part {
  int R, C, br, bc;
};

// out (nrows x p, ld ldo, row-major in smem or strided) = Aop (nrows x K) B (K x p),
// A element (i, kk) at a[i * ai + kk * ak], B element (kk, j) at b[kk * bk + j].
// C (nrows x p) = A (nrows x K) B (K x p) from shared memory on the FP64
// tensor pipe: mma.sync m16n8k4 f64 (DMMA).  A element (i, kk) at
// a[i * ai + kk * ak], B element (kk, j) at b[kk * bk + j]; C element (i, j)
// stored to dst[j * ld_j + i * ld_i].  A warp owns one 16-row tile and all
// p / 8 column tiles of it (the A fragment is loaded once per k-step for
// all of them): 2 + p / 8 shared loads per p / 8 MMAs of 512 FMAs each --
// the FMA-per-load ratio the CUDA-core version lacked.  Out-of-range rows /
// columns / k are read as zero.
template <int NTMAX>
__device__ __forceinline__ void v4_block_gemm(const double* __restrict__ a, int ai, int ak, const double* __restrict__ b,
                                              int bk, int nrows, int K, int p, double* __restrict__ dst,
                                              int64_t ld_j, int64_t ld_i) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int ntiles = (p + 7) / 8;
  for (int mt = warp; mt * 16 < nrows; mt += nwarps) {
    const int m0 = mt * 16;
    double acc[NTMAX][4];
#pragma unroll
    for (int n = 0; n < NTMAX; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[n][q] = 0.0;
    const int r0 = m0 + g, r1 = m0 + g + 8;
    const bool v0 = r0 < nrows, v1 = r1 < nrows;
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int kk = k0 + t;
      const bool kv = kk < K;
      const double a0 = (v0 && kv) ? a[r0 * ai + kk * ak] : 0.0;
      const double a1 = (v1 && kv) ? a[r1 * ai + kk * ak] : 0.0;
#pragma unroll
      for (int n = 0; n < NTMAX; ++n) {
        if (n < ntiles) {
          const int col = n * 8 + g;
          const double b0 = (kv && col < p) ? b[kk * bk + col] : 0.0;
          asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                       : "+d"(acc[n][0]), "+d"(acc[n][1]), "+d"(acc[n][2]), "+d"(acc[n][3])
                       : "d"(a0), "d"(a1), "d"(b0));
        }
      }
    }
#pragma unroll
    for (int n = 0; n < NTMAX; ++n) {
      if (n < ntiles) {
        const int c0 = n * 8 + 2 * t, c1 = c0 + 1;
        if (v0 && c0 < p) dst[c0 * ld_j + r0 * ld_i] = acc[n][0];
        if (v0 && c1 < p) dst[c1 * ld_j + r0 * ld_i] = acc[n][1];
        if (v1 && c0 < p) dst[c0 * ld_j + r1 * ld_i] = acc[n][2];
        if (v1 && c1 < p) dst[c1 * ld_j + r1 * ld_i] = acc[n][3];
      }
    }
  }
}

// Op[i * p + j] = M[i + j * ldm] for i < rows, j < p (L2 loads, 8 in flight)
__device__ __forceinline__ void stage_op(const double* __restrict__ M, int64_t ldm, int rows, int p,
                                         double* __restrict__ Op, int pst) {
  const int tot = rows * p, nt = blockDim.x;
  for (int e0 = threadIdx.x; e0 < tot; e0 += 8 * nt) {
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = e0 + t * nt;
      v[t] = e < tot ? __ldcg(&M[(e % rows) + (int64_t)(e / rows) * ldm]) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int e = e0 + t * nt;
      if (e < tot) Op[(e % rows) * pst + e / rows] = v[t];
    }
  }
}

// sum_{q < n} x[q * stride] in q order; loads issued 8 at a time (L2,
// bypassing L1: the partials were written by other CTAs since the last
// barrier), so a long sum costs n / 8 round trips, not n
__device__ __forceinline__ double sum_strided(const double* __restrict__ x, int64_t stride, int n) {
  double s = 0.0;
  int q = 0;
  for (; q + 8 <= n; q += 8) {
    double v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) v[t] = __ldcg(x + (int64_t)(q + t) * stride);
#pragma unroll
    for (int t = 0; t < 8; ++t) s += v[t];
  }
  for (; q < n; ++q) s += __ldcg(x + (int64_t)q * stride);
  return s;
}

__global__ void __launch_bounds__(kV4T, 1)
richardson_v4(int k, int c, int p, const double* __restrict__ S, int64_t lds, const double* __restrict__ P,
              int64_t ldp, int l, double* __restrict__ X, int64_t ldx, double* __restrict__ T, int64_t ldt,
              double* __restrict__ ws, V4Part pt) {
  extern __shared__ __align__(16) double v4s[];
  cg::grid_group grid = cg::this_grid();
  const int nblk = pt.R * pt.C;
  const int b = blockIdx.x;
  const bool own = b < nblk;
  const int rb = own ? b / pt.C : 0, cb = own ? b % pt.C : 0;
  const int r0 = rb * pt.br, a0 = cb * pt.bc;
  const int nr = own ? max(0, min(pt.br, k - r0)) : 0, na = own ? max(0, min(pt.bc, c - a0)) : 0;
  // strides padded for 16-byte vector loads: even block column stride, row
  // stride of the staged operand a multiple of 4 doubles
  const int bst = (pt.br + 1) & ~1, pst = (p + 3) & ~3;
  double* Sb = v4s;                                  // [a][r], stride bst (column-major block)
  double* Op = v4s + (((int64_t)bst * pt.bc + 3) & ~3);  // X_cb as [a][j] or T_r as [r][j], stride pst
  double* wsA = ws;                                   // [cb][j][r]: C * p * k
  double* wsB = ws + (int64_t)pt.C * p * k;           // [rb][j][a]: R * p * c
  // the block of S, once
  for (int e = threadIdx.x; e < nr * na; e += kV4T) {
    const int r = e % nr, a = e / nr;
    cpa8(&Sb[a * bst + r], &S[(r0 + r) + (int64_t)(a0 + a) * lds]);
  }
  cpa_commit();
  KDIM_MARK(0);
  const int64_t nthreads = (int64_t)gridDim.x * kV4T, gtid = (int64_t)b * kV4T + threadIdx.x;
  for (int sweep = 0; sweep < l; ++sweep) {
    if (sweep > 0) {
      // A: partial T = S_(r,cb) X_cb
      // X_cb (written by other CTAs: L2 loads), 8 loads in flight per thread
      stage_op(X + a0, ldx, na, p, Op, pst);
      cpa_wait<0>();
      __syncthreads();
      KDIM_MARK(8 * sweep + 1);
      if (nr > 0)
        v4_block_gemm<8>(Sb, 1, bst, Op, pst, nr, na, p, wsA + (int64_t)cb * p * k + r0, k, 1);
      KDIM_MARK(8 * sweep + 2);
      grid.sync();
      KDIM_MARK(8 * sweep + 3);
      for (int64_t e = gtid; e < (int64_t)k * p; e += nthreads) {
        const int r = (int)(e % k), j = (int)(e / k);
        const double sx = sum_strided(wsA + (int64_t)j * k + r, (int64_t)p * k, pt.C);
        T[r + (int64_t)j * ldt] = P[r + (int64_t)j * ldp] - sx;
      }
      grid.sync();
      KDIM_MARK(8 * sweep + 4);
    }
    // B: partial X = S_(r,cb)^T T_r (sweep 0: T = P)
    const double* Tin = sweep == 0 ? P : T;
    const int64_t ldtin = sweep == 0 ? ldp : ldt;
    stage_op(Tin + r0, ldtin, nr, p, Op, pst);
    cpa_wait<0>();
    __syncthreads();
    KDIM_MARK(8 * sweep + 5);
    if (na > 0)
      v4_block_gemm<8>(Sb, bst, 1, Op, pst, na, nr, p, wsB + (int64_t)rb * p * c + a0, c, 1);
    KDIM_MARK(8 * sweep + 6);
    grid.sync();
    KDIM_MARK(8 * sweep + 7);
    for (int64_t e = gtid; e < (int64_t)c * p; e += nthreads) {
      const int a = (int)(e % c), j = (int)(e / c);
      const double st = sum_strided(wsB + (int64_t)j * c + a, (int64_t)p * c, pt.R);
      double* xp = X + a + (int64_t)j * ldx;
      *xp = sweep == 0 ? st : *xp + st;
    }
    if (sweep + 1 < l) grid.sync();
    KDIM_MARK(8 * sweep + 8);
    __syncthreads();
  }
}

// ============================ sketched CholQR ===============================
// Cholesky of the p x p matrix in shared memory (upper, right-looking, dpotrf
// semantics): returns 0 or the 1-based column of the first pivot <= 0 / NaN.
__device__ int chol_smem(double* Sm, int p, int* bad_sh) {
  if (threadIdx.x == 0) *bad_sh = 0;
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double d = Sm[j + j * p];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) *bad_sh = j + 1;
      break;
    }
    const double r = sqrt(d);
    for (int cc = j + 1 + threadIdx.x; cc < p; cc += blockDim.x) Sm[j + cc * p] /= r;
    __syncthreads();
    if (threadIdx.x == 0) Sm[j + j * p] = r;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
    for (int b = j + 1 + ty; b < p; b += ny) {
      const double sjb = Sm[j + b * p];
      for (int a = j + 1 + tx; a <= b; a += 32) Sm[a + b * p] -= Sm[j + a * p] * sjb;
    }
    __syncthreads();
  }
  __syncthreads();
  return *bad_sh;
}

// G = S'^T S' (8-row items over the p columns, K = k), grid barrier; CTA 0
// factors G; grid barrier; every CTA solves its rows of Sout = S' R^{-1}.
template <int PB>
__global__ void __launch_bounds__(256, 1)
cholqr_v3(int k, int p, const double* __restrict__ Sp, int64_t lds, double* __restrict__ R, int64_t ldr,
          double* __restrict__ Sout, int64_t ldso, int* __restrict__ info, double* __restrict__ ws) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ItemSmem<PB, 8>& sm = *reinterpret_cast<ItemSmem<PB, 8>*>(smraw);
  double* smd = reinterpret_cast<double*>(smraw);
  __shared__ int bad;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  double* Gg = ws;              // p x p (ld p)
  double* Rg = ws + p * p;      // R (p x p) + 1 / diag
  for (int t = blockIdx.x; t < (p + 7) / 8; t += G) {
    const int mrows = min(8, p - 8 * t);
    tile_item<PB, 8, true>(Sp + (int64_t)8 * t * lds, lds, Sp, lds, 0, mrows, p, k, sm);
    for (int e = threadIdx.x; e < mrows * p; e += 256) {
      const int i = e % mrows, j = e / mrows;
      Gg[(8 * t + i) + j * p] = sm.red[0][j * 8 + i];
    }
    __syncthreads();
  }
  grid.sync();
  if (blockIdx.x == 0) {
    double* Gm = smd;
    for (int e = threadIdx.x; e < p * p; e += 256) {
      const int i = e % p, j = e / p;
      Gm[e] = i <= j ? __ldcg(&Gg[e]) : 0.0;
    }
    __syncthreads();
    const int b = chol_smem(Gm, p, &bad);
    for (int e = threadIdx.x; e < p * p; e += 256) {
      const int i = e % p, j = e / p;
      const double v = i <= j ? Gm[e] : 0.0;
      R[i + (int64_t)j * ldr] = v;
      Rg[e] = v;
    }
    for (int j = threadIdx.x; j < p; j += 256) Rg[p * p + j] = 1.0 / Gm[j + j * p];
    if (threadIdx.x == 0) *info = b;
  }
  grid.sync();
  // Sout = S' R^{-1}: one row per thread, fp64, l ascending (rb_trsm_right's
  // order: t = fma(-x_l, R_lj, t), x_j = t * (1 / R_jj))
  double* Rs = smd;
  for (int e = threadIdx.x; e < p * p + p; e += 256) Rs[e] = __ldcg(&Rg[e]);
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x; r < k; r += (int64_t)G * 256) {
    double x[PB];
#pragma unroll
    for (int j = 0; j < PB; ++j) x[j] = j < p ? Sp[r + (int64_t)j * lds] : 0.0;
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      if (j < p) {
        double t = x[j];
#pragma unroll
        for (int l2 = 0; l2 < j; ++l2) t = fma(-x[l2], Rs[l2 + j * p], t);
        x[j] = t * Rs[p * p + j];
      }
    }
#pragma unroll
    for (int j = 0; j < PB; ++j)
      if (j < p) Sout[r + (int64_t)j * ldso] = x[j];
  }
}

// Upper Cholesky of the p x p matrix Gm (column-major, smem) with ONE
// block barrier per column: at step j every thread reads the (final) row j,
// forms the scaled entries R_ja = G_ja / R_jj on the fly and updates its
// trailing entries G_ab -= R_ja R_jb (j < a <= b) -- the operations and
// per-element order of chol_smem, so the same bits -- while the owners of
// row j write R_jc into Rm (a separate array, no read/write overlap).
// Returns 0 or the 1-based column of the first pivot <= 0 / NaN (dpotrf).
__device__ int chol_onebar(double* Gm, double* Rm, int p, int* bad_sh) {
  if (threadIdx.x == 0) *bad_sh = 0;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) Rm[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    const double d = Gm[j + j * p];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) *bad_sh = j + 1;
      break;
    }
    const double r = sqrt(d);
    const int m = p - j - 1;  // trailing order
    for (int c = j + threadIdx.x; c < p; c += blockDim.x) Rm[j + c * p] = c == j ? r : Gm[j + c * p] / r;
    // trailing upper entries (a, b), j < a <= b < p, enumerated column by column
    for (int e = threadIdx.x; e < m * (m + 1) / 2; e += blockDim.x) {
      int bb = (int)((sqrtf(8.f * e + 1.f) - 1.f) * 0.5f);  // column index within the trailing block
      while ((bb + 1) * (bb + 2) / 2 <= e) ++bb;
      while (bb * (bb + 1) / 2 > e) --bb;
      const int aa = e - bb * (bb + 1) / 2;
      const int A = j + 1 + aa, B = j + 1 + bb;
      Gm[A + B * p] -= (Gm[j + A * p] / r) * (Gm[j + B * p] / r);
    }
    __syncthreads();
  }
  __syncthreads();
  return *bad_sh;
}

// x <- x R^{-1} for one row (R in smem, ld ldr; inv[j] = 1 / R_jj), the
// order of rb_trsm_right's tri_solve_row: per column, t = x_j, then
// t = fma(-x_l, R_lj, t) for l ascending, x_j = t * inv_j; CH columns at a
// time as independent chains (each keeps its own l-ascending order).
template <int PB, int CH>
__device__ __forceinline__ void tri_solve_smem(double (&x)[PB], int p, const double* Rm, int ldr, const double* inv) {
#pragma unroll
  for (int j = 0; j < PB; j += CH) {
    if (j + CH <= PB && j + CH <= p) {
      double s[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) s[c] = x[j + c];
#pragma unroll
      for (int l = 0; l < j; ++l)
#pragma unroll
        for (int c = 0; c < CH; ++c) s[c] = fma(-x[l], Rm[l + (j + c) * ldr], s[c]);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        x[j + c] = s[c] * inv[j + c];
#pragma unroll
        for (int c2 = c + 1; c2 < CH; ++c2) s[c2] = fma(-x[j + c], Rm[j + c + (j + c2) * ldr], s[c2]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int jj = j + c;
        if (jj < PB && jj < p) {
          double t = x[jj];
#pragma unroll
          for (int l = 0; l < jj; ++l) t = fma(-x[l], Rm[l + jj * ldr], t);
          x[jj] = t * inv[jj];
        }
      }
    }
  }
}

// v4: the Gram split over K across CTAs (each loads its row slice of S' once,
// 8 loads in flight per thread), a distributed fixed-order reduction of the
// partials, the factorization on CTA 0, then the row solves.
template <int PB>
__global__ void __launch_bounds__(256, 1)
cholqr_v4(int k, int p, const double* __restrict__ Sp, int64_t lds, double* __restrict__ R, int64_t ldr,
          double* __restrict__ Sout, int64_t ldso, int* __restrict__ info, double* __restrict__ ws, int ks) {
  extern __shared__ __align__(16) double c4s[];
  __shared__ int bad;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  const int pp = p * p;
  double* part = ws;                       // [G][p * p] (upper triangle used)
  double* Gg = ws + (int64_t)G * pp;       // reduced G
  double* Rg = Gg + pp;                    // R + 1 / diag
  KDIM_MARK(100);
  // phase 1: this CTA's rows [q ks, (q + 1) ks) of S' -> smem [r][j], then the upper triangle
  {
    const int r0 = blockIdx.x * ks, nr = max(0, min(ks, k - r0));
    double* sl = c4s;  // nr x p, row-major
    stage_op(Sp + r0, lds, nr, p, sl, p);
    __syncthreads();
    KDIM_MARK(110);
    // the slice's Gram on the FP64 tensor pipe (full p x p; the upper triangle is used)
    v4_block_gemm<8>(sl, 1, p, sl, p, p, nr, p, part + (int64_t)blockIdx.x * pp, p, 1);
  }
  KDIM_MARK(101);
  grid.sync();
  KDIM_MARK(102);
  // phase 2: G = sum over CTAs (CTA order), upper triangle
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < pp; e += (int64_t)G * 256) {
    const int i = (int)(e % p), j = (int)(e / p);
    if (i <= j) Gg[e] = sum_strided(part + e, pp, G);
  }
  grid.sync();
  KDIM_MARK(103);
  if (blockIdx.x == 0) {
    double* Gm = c4s;
    for (int e = threadIdx.x; e < pp; e += 256) {
      const int i = e % p, j = e / p;
      Gm[e] = i <= j ? __ldcg(&Gg[e]) : 0.0;
    }
    __syncthreads();
    double* Rm = c4s + pp;
    const int b = chol_onebar(Gm, Rm, p, &bad);
    for (int e = threadIdx.x; e < pp; e += 256) {
      const int i = e % p, j = e / p;
      const double v = i <= j ? Rm[e] : 0.0;
      R[i + (int64_t)j * ldr] = v;
      Rg[e] = v;
    }
    for (int j = threadIdx.x; j < p; j += 256) Rg[pp + j] = 1.0 / Rm[j + j * p];
    if (threadIdx.x == 0) *info = b;
  }
  KDIM_MARK(104);
  grid.sync();
  KDIM_MARK(105);
  // Sout = S' R^{-1}: one row per thread, fp64, l ascending (rb_trsm_right's
  // order: t = fma(-x_l, R_lj, t), x_j = t * (1 / R_jj))
  double* Rs = c4s;
  for (int e = threadIdx.x; e < pp + p; e += 256) Rs[e] = __ldcg(&Rg[e]);
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * 256 + threadIdx.x; r < k; r += (int64_t)G * 256) {
    double x[PB];
#pragma unroll
    for (int j = 0; j < PB; ++j) x[j] = j < p ? Sp[r + (int64_t)j * lds] : 0.0;
    tri_solve_smem<PB, (PB < 32 ? 4 : 2)>(x, p, Rs, p, Rs + pp);
#pragma unroll
    for (int j = 0; j < PB; ++j)
      if (j < p) Sout[r + (int64_t)j * ldso] = x[j];
  }
  KDIM_MARK(106);
}

// ============================ certification =================================
// out[0] = ||I - S^T S||_F^2, out[1] = ||P - S R||_F^2, out[2] = ||P||_F^2
// (rbgs.py:428-443); S, P k x m, R m x m.  Tiles of 64 x 64; the split-K
// partials are summed in split order, then the squares in a fixed
// two-stage order.
__global__ void __launch_bounds__(kKT)
certify_coop(int k, int m, const double* __restrict__ S, int64_t lds, const double* __restrict__ P, int64_t ldp,
             const double* __restrict__ R, int64_t ldr, double* __restrict__ out, double* __restrict__ ws) {
  extern __shared__ __align__(16) double smem[];
  __shared__ double red[kKT / 32];
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x;
  constexpr int PB = 64;
  const int mt = (m + kTM - 1) / kTM, kt = (k + kTM - 1) / kTM;
  const int tilesG = mt * mt, tilesE = kt * mt;
  const int splitsG = splits_for(tilesG, k, G), splitsE = splits_for(tilesE, m, G);
  double* wsG = ws;
  double* wsE = ws + (int64_t)tilesG * splitsG * (kTM * PB);
  double* part = wsE + (int64_t)tilesE * splitsE * (kTM * PB);  // [3][G]
  for (int it = blockIdx.x; it < tilesG * splitsG + tilesE * splitsE; it += G) {
    double acc[2][PB / 8];
    if (it < tilesG * splitsG) {  // (S^T S) tile (ti, tj), split s over k
      const int t = it % tilesG, s = it / tilesG;
      const int ti = t % mt, tj = t / mt;
      int64_t kb, ke;
      split_range(k, splitsG, s, kb, ke);
      tile_gemm<PB, true>(S, lds, S + (int64_t)tj * kTM * lds, lds, ti * kTM, min(kTM, m - ti * kTM),
                          min(kTM, m - tj * kTM), kb, ke, acc, smem);
      store_partial<PB>(wsG + (int64_t)it * (kTM * PB), acc);
    } else {  // (S R) tile (ti over k, tj over m), split s over m
      const int i2 = it - tilesG * splitsG;
      const int t = i2 % tilesE, s = i2 / tilesE;
      const int ti = t % kt, tj = t / kt;
      int64_t kb, ke;
      split_range(m, splitsE, s, kb, ke);
      tile_gemm<PB, false>(S, lds, R + (int64_t)tj * kTM * ldr, ldr, ti * kTM, min(kTM, k - ti * kTM),
                           min(kTM, m - tj * kTM), kb, ke, acc, smem);
      store_partial<PB>(wsE + (int64_t)i2 * (kTM * PB), acc);
    }
  }
  grid.sync();
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int64_t nthreads = (int64_t)G * kKT, gtid = (int64_t)blockIdx.x * kKT + threadIdx.x;
  for (int64_t e = gtid; e < (int64_t)m * m; e += nthreads) {
    const int i = (int)(e % m), j = (int)(e / m);
    const int t = (i / kTM) + (j / kTM) * mt;
    const double g = sum_splits<PB>(wsG, tilesG, splitsG, t, i % kTM, j % kTM);
    const double d = (i == j ? 1.0 : 0.0) - g;
    a0 += d * d;
  }
  for (int64_t e = gtid; e < (int64_t)k * m; e += nthreads) {
    const int r = (int)(e % k), j = (int)(e / k);
    const int t = (r / kTM) + (j / kTM) * kt;
    const double sr = sum_splits<PB>(wsE, tilesE, splitsE, t, r % kTM, j % kTM);
    const double pv = P[r + (int64_t)j * ldp];
    const double d = pv - sr;
    a1 += d * d;
    a2 += pv * pv;
  }
  a0 = block_sum(a0, red);
  a1 = block_sum(a1, red);
  a2 = block_sum(a2, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = a0;
    part[G + blockIdx.x] = a1;
    part[2 * G + blockIdx.x] = a2;
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x < 3) {
    double s = 0.0;
    for (int q = 0; q < G; ++q) s += part[threadIdx.x * G + q];
    out[threadIdx.x] = s;
  }
}

// ============================ generic GEMM ==================================
// C = alpha op(A) B + beta C (op = transpose when tA), type T in and out
// (double: binary64; float: the binary32 Step-2 solvers of unique-coarse
// mode, rbgs.py:144-212 with prec.dtype = float32).  128 x 64 tiles, 256
// threads, 8 x 4 accumulators per thread fed by LDS.128; split over K into
// the workspace (summed in split order by gemm_reduce) when the tile grid is
// too small to fill the GPU, else the epilogue is applied in place.
constexpr int kGM = 128, kGN = 64, kGK = 16;

template <typename T, bool TRANS_A>
__global__ void __launch_bounds__(256)
gemm_tiles(int m, int n, int64_t K, const T* __restrict__ A, int64_t lda, const T* __restrict__ B, int64_t ldb,
           int64_t chunk, T alpha, T beta, T* __restrict__ C, int64_t ldc, T* __restrict__ ws, int upper) {
  using V4 = typename std::conditional<sizeof(T) == 8, double4, float4>::type;
  // double-buffered tiles: the next K step is fetched into registers while
  // the current one is multiplied (one barrier per step)
  // rows padded by 4 entries: the K-fastest stores of a fetched tile (16
  // consecutive k per row of op(A) / B) would otherwise all hit one bank
  extern __shared__ __align__(32) unsigned char gemm_smem[];
  T (*sA)[kGK][kGM + 4] = reinterpret_cast<T (*)[kGK][kGM + 4]>(gemm_smem);
  T (*sB)[kGK][kGN + 4] = reinterpret_cast<T (*)[kGK][kGN + 4]>(gemm_smem + 2 * kGK * (kGM + 4) * sizeof(T));
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;  // rows 8 ty.., cols 4 tx..
  const int m0 = blockIdx.x * kGM, n0 = blockIdx.y * kGN;
  // symmetric product (A^T A): tiles entirely below the diagonal are not formed
  if (upper && m0 >= n0 + kGN) return;
  const int64_t kb = (int64_t)blockIdx.z * chunk, ke = min(K, kb + chunk);
  constexpr int kEA = kGK * kGM / 256, kEB = kGK * kGN / 256;
  T ra[kEA], rb[kEB];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int u = 0; u < kEA; ++u) {
      const int e = tid + 256 * u;
      int i, kk;
      if (TRANS_A) { kk = e % kGK; i = e / kGK; } else { i = e % kGM; kk = e / kGM; }
      const int64_t kg = k0 + kk;
      ra[u] = (m0 + i < m && kg < ke) ? (TRANS_A ? A[kg + (int64_t)(m0 + i) * lda] : A[(m0 + i) + kg * lda]) : T(0);
    }
#pragma unroll
    for (int u = 0; u < kEB; ++u) {
      const int e = tid + 256 * u;
      const int kk = e % kGK, jj = e / kGK;
      const int64_t kg = k0 + kk;
      rb[u] = (n0 + jj < n && kg < ke) ? B[kg + (int64_t)(n0 + jj) * ldb] : T(0);
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int u = 0; u < kEA; ++u) {
      const int e = tid + 256 * u;
      int i, kk;
      if (TRANS_A) { kk = e % kGK; i = e / kGK; } else { i = e % kGM; kk = e / kGM; }
      sA[buf][kk][i] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < kEB; ++u) {
      const int e = tid + 256 * u;
      sB[buf][e % kGK][e / kGK] = rb[u];
    }
  };
  T acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);
  int buf = 0;
  if (kb < ke) {
    fetch(kb);
    stash(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += kGK) {
    const bool more = k0 + kGK < ke;
    if (more) fetch(k0 + kGK);
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      T a[8], b[4];
      const V4 a0 = *reinterpret_cast<const V4*>(&sA[buf][kk][8 * ty]);
      const V4 a1 = *reinterpret_cast<const V4*>(&sA[buf][kk][8 * ty + 4]);
      const V4 b0 = *reinterpret_cast<const V4*>(&sB[buf][kk][4 * tx]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[q][t] = fma(a[q], b[t], acc[q][t]);
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  // a thread's 8 rows are contiguous: whole-vector stores (full sectors)
  // when the tile is interior and C is aligned -- the tall n x 240 outputs
  // of the GMRES corrections are write-bound otherwise
  T* Cd = ws ? ws + (int64_t)blockIdx.z * m * n : C;
  const int64_t ldd = ws ? m : ldc;
  const bool vec = m0 + kGM <= m && ldd % 4 == 0 && ((uintptr_t)Cd % (4 * sizeof(T))) == 0 &&
                   (ws || beta == T(0));
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int jj = n0 + 4 * tx + t;
    if (jj >= n) continue;
    const T sc = ws ? T(1) : alpha;
    if (vec) {
      V4 v0, v1;
      v0.x = sc * acc[0][t]; v0.y = sc * acc[1][t]; v0.z = sc * acc[2][t]; v0.w = sc * acc[3][t];
      v1.x = sc * acc[4][t]; v1.y = sc * acc[5][t]; v1.z = sc * acc[6][t]; v1.w = sc * acc[7][t];
      V4* dst = reinterpret_cast<V4*>(Cd + (m0 + 8 * ty) + (int64_t)jj * ldd);
      dst[0] = v0;
      dst[1] = v1;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int i = m0 + 8 * ty + q;
        if (i < m) {
          T* c = Cd + i + (int64_t)jj * ldd;
          if (ws) *c = acc[q][t];
          else *c = beta == T(0) ? alpha * acc[q][t] : alpha * acc[q][t] + beta * *c;
        }
      }
    }
  }
}

// Tall binary64 product C (M x N) = alpha A (M x K) B (K x N) + beta C for
// M >> N, K (the GMRES corrections U = Q Z, krylov.py:247-262: 1.7e7 x 244
// times 244 x 240) on the FP64 tensor pipe: a CTA owns 128 rows x 64 columns,
// a warp 16 rows and all eight 8-column tiles (mma.sync m16n8k4 f64: one A
// fragment per k-step serves them); A and B chunks of 32 k are staged in
// shared memory with pitches (136, 36) that make staging stores and fragment
// loads conflict-free.  k ascending per output: deterministic.
constexpr int kNNM = 128, kNNN = 64, kNNK = 32, kNNPA = 136, kNNPB = 36;

__global__ void __launch_bounds__(256, 2)
gemm_nn_dmma(int64_t M, int N, int K, double alpha, const double* __restrict__ A, int64_t lda,
             const double* __restrict__ B, int64_t ldb, double beta, double* __restrict__ C, int64_t ldc) {
  extern __shared__ double nn_sm[];
  double* sA = nn_sm;                    // [kNNK][kNNPA]: (k, row)
  double* sB = nn_sm + kNNK * kNNPA;     // [kNNN][kNNPB]: (col, k)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int64_t m0 = (int64_t)blockIdx.x * kNNM;
  const int n0 = blockIdx.y * kNNN;
  double acc[8][4];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < K; k0 += kNNK) {
    __syncthreads();
    for (int e = tid; e < kNNK * kNNM; e += 256) {
      const int i = e % kNNM, kk = e / kNNM;
      sA[kk * kNNPA + i] = (m0 + i < M && k0 + kk < K) ? A[(m0 + i) + (int64_t)(k0 + kk) * lda] : 0.0;
    }
    for (int e = tid; e < kNNK * kNNN; e += 256) {
      const int kk = e % kNNK, j = e / kNNK;
      sB[j * kNNPB + kk] = (n0 + j < N && k0 + kk < K) ? B[(k0 + kk) + (int64_t)(n0 + j) * ldb] : 0.0;
    }
    __syncthreads();
    const int r = warp * 16 + g;
#pragma unroll
    for (int ks = 0; ks < kNNK; ks += 4) {
      const double a0 = sA[(ks + t) * kNNPA + r];
      const double a1 = sA[(ks + t) * kNNPA + r + 8];
#pragma unroll
      for (int nn = 0; nn < 8; ++nn) {
        const double b0 = sB[(nn * 8 + g) * kNNPB + ks + t];
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[nn][0]), "+d"(acc[nn][1]), "+d"(acc[nn][2]), "+d"(acc[nn][3])
                     : "d"(a0), "d"(a1), "d"(b0));
      }
    }
  }
#pragma unroll
  for (int nn = 0; nn < 8; ++nn) {
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int64_t i = m0 + warp * 16 + g + (h >> 1) * 8;
      const int j = n0 + nn * 8 + 2 * t + (h & 1);
      if (i < M && j < N) {
        double* c = C + i + (int64_t)j * ldc;
        *c = beta == 0.0 ? alpha * acc[nn][h] : alpha * acc[nn][h] + beta * *c;
      }
    }
  }
}

template <typename T>
__global__ void gemm_reduce(const T* __restrict__ ws, int splits, int m, int n, T alpha, T beta, T* __restrict__ C,
                            int64_t ldc, int upper) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)m * n;
  if (e >= tot) return;
  if (upper && (int)(e % m) / kGM * kGM >= (int)(e / m) / kGN * kGN + kGN) return;  // tile not formed
  T s = T(0);
  for (int q = 0; q < splits; ++q) s += ws[(int64_t)q * tot + e];
  const int i = (int)(e % m), j = (int)(e / m);
  T* c = C + i + (int64_t)j * ldc;
  *c = beta == T(0) ? alpha * s : alpha * s + beta * *c;
}

template <typename T>
int gemm_generic(int tA, int m, int n, int64_t K, T alpha, const T* A, int64_t lda, const T* B, int64_t ldb, T beta,
                 T* C, int64_t ldc, void* ws, size_t wsb, cudaStream_t st, const char* what, int upper = 0) {
  if (m == 0 || n == 0) return RB_OK;
  if constexpr (std::is_same<T, double>::value) {
    // tall outputs only: the k-dimensional products keep their own summation order
    static const int nn_dmma = getenv("RB_GEMM_DMMA") ? atoi(getenv("RB_GEMM_DMMA")) : 1;
    if (nn_dmma && !tA && !upper && m >= 65536 && K >= 1 && K <= 4096) {
      const size_t smem = (size_t)(kNNK * kNNPA + kNNN * kNNPB) * sizeof(double);
      cudaFuncSetAttribute(gemm_nn_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const dim3 grid((unsigned)((m + kNNM - 1) / kNNM), (unsigned)((n + kNNN - 1) / kNNN));
      RB_KLAUNCH gemm_nn_dmma<<<grid, 256, smem, st>>>((int64_t)m, n, (int)K, (double)alpha, (const double*)A, lda,
                                                       (const double*)B, ldb, (double)beta, (double*)C, ldc);
      return check_launch(what);
    }
  }
  const int mt = (m + kGM - 1) / kGM, nt = (n + kGN - 1) / kGN;
  const int64_t tiles = (int64_t)mt * nt;
  const int64_t want = 2 * (int64_t)sm_count();
  int64_t splits = 1;
  if (tiles < want && K > 4 * kGK) splits = std::min<int64_t>((want + tiles - 1) / tiles, (K + 4 * kGK - 1) / (4 * kGK));
  const size_t per = (size_t)m * n * sizeof(T);
  if (splits > 1 && (!ws || splits * per > wsb)) splits = ws ? std::max<int64_t>(1, (int64_t)(wsb / per)) : 1;
  splits = std::min<int64_t>(splits, 65535);
  int64_t chunk = K > 0 ? (K + splits - 1) / splits : 0;
  chunk = (chunk + kGK - 1) / kGK * kGK;
  if (chunk == 0) chunk = kGK;
  splits = std::max<int64_t>(1, (K + chunk - 1) / chunk);
  T* part = splits > 1 ? (T*)ws : nullptr;
  RB_REQUIRE(mt <= INT32_MAX && nt <= 65535, "%s: too large", what);
  const dim3 grid((unsigned)mt, (unsigned)nt, (unsigned)splits);
  const size_t smem = 2 * kGK * (kGM + 4 + kGN + 4) * sizeof(T);
  if (tA) {
    cudaFuncSetAttribute(gemm_tiles<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    RB_KLAUNCH gemm_tiles<T, true><<<grid, 256, smem, st>>>(m, n, K, A, lda, B, ldb, chunk, alpha, beta, C, ldc, part,
                                                            upper);
  } else {
    cudaFuncSetAttribute(gemm_tiles<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    RB_KLAUNCH gemm_tiles<T, false><<<grid, 256, smem, st>>>(m, n, K, A, lda, B, ldb, chunk, alpha, beta, C, ldc, part,
                                                             upper);
  }
  if (part) RB_KLAUNCH gemm_reduce<T><<<ceil_div((int64_t)m * n, 256), 256, 0, st>>>(part, (int)splits, m, n, alpha,
                                                                                     beta, C, ldc, upper);
  return check_launch(what);
}

// ---- launch helpers -----------------------------------------------------------
template <typename K>
int coop_launch(K kern, size_t smem, void** args, cudaStream_t st, int max_grid, int* grid_out, const char* what,
                int nthreads = kKT) {
  static int dev_cached = -1;
  (void)dev_cached;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nthreads, smem);
  RB_REQUIRE(per_sm >= 1, "%s: kernel does not fit an SM", what);
  int grid = std::min(max_grid, sm_count() * std::min(per_sm, 2));
  grid = std::max(grid, 1);
  *grid_out = grid;
  ++g_launches;
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(nthreads), args, smem, st);
  if (e != cudaSuccess) {
    set_error("%s: cooperative launch failed: %s", what, cudaGetErrorString(e));
    return RB_ECUDA;
  }
  return check_launch(what);
}

}  // namespace

// Workspace of the cooperative k-dimensional kernels (upper bound): split-K
// partial tiles for a grid of 2 CTAs per SM plus the output tiles.
size_t kdim_ws_bytes(int k, int m) {
  const size_t grid = 4 * (size_t)sm_count();
  const size_t tiles = (size_t)((k + kTM - 1) / kTM + 1) * ((m + kTM - 1) / kTM + 1);
  return (grid + tiles + 4) * (size_t)kTM * 64 * sizeof(double) + 3 * grid * sizeof(double) + 4096;
}

// Block grid of S for richardson_v4: C column blocks, R = G / C row blocks,
// C chosen so the blocks are about square (balanced partial reductions);
// nullopt-like (R = 0) when a block does not fit the shared-memory budget.
static size_t v4_smem(int br, int bc, int p) {
  const size_t bst = (size_t)((br + 1) & ~1), pst = (size_t)((p + 3) & ~3);
  return (((bst * bc + 3) & ~(size_t)3) + (size_t)std::max(br, bc) * pst) * sizeof(double);
}

static V4Part v4_partition(int k, int c, int p, int G) {
  V4Part best{0, 0, 0, 0};
  size_t best_cost = (size_t)-1;
  for (int C = 1; C <= std::min(c, G); ++C) {
    const int R = std::min(k, G / C);
    if (R < 1) break;
    const int br = (k + R - 1) / R, bc = (c + C - 1) / C;
    const size_t smem = v4_smem(br, bc, p);
    if (smem > (size_t)kV4Smem) continue;
    // per-sweep cost model: block FMAs (both phases) + reduction loads per thread
    const size_t cost = 2 * (size_t)br * bc * p / 64 + ((size_t)k * C + (size_t)c * R) * p / ((size_t)G * kV4T) * 400;
    if (cost < best_cost) {
      best_cost = cost;
      best = V4Part{(k + br - 1) / br, (c + bc - 1) / bc, br, bc};
    }
  }
  return best;
}

int ls_richardson(int k, int c, int p, const double* S, int64_t lds, const double* P, int64_t ldp, int l, double* X,
                  int64_t ldx, double* T, int64_t ldt, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(k >= 1 && c >= 1 && p >= 1 && p <= 64 && l >= 1 && S && P && X && T && lds >= k && ldp >= k &&
                 ldx >= c && ldt >= k,
             "rb_ls_richardson: bad args (k=%d c=%d p=%d l=%d)", k, c, p, l);
  const int G = sm_count();
  V4Part pt = v4_partition(k, c, p, G);
  if (pt.R > 0) {
    const size_t need = ((size_t)pt.C * p * k + (size_t)pt.R * p * c) * sizeof(double);
    RB_REQUIRE(ws && wsb >= need, "rb_ls_richardson: workspace too small (%zu < %zu)", wsb, need);
    int grid = 0;
    void* args[] = {&k, &c, &p, (void*)&S, &lds, (void*)&P, &ldp, &l, &X, &ldx, &T, &ldt, &ws, &pt};
    const size_t smem = v4_smem(pt.br, pt.bc, p);
    return coop_launch(richardson_v4, smem, args, st, pt.R * pt.C, &grid, "rb_ls_richardson", kV4T);
  }
  // S too large for the grid's shared memory: full-K tile items
  const int items = std::max(l > 1 ? (k + 15) / 16 : 1, (c + 7) / 8);
  const int G3 = std::max(1, std::min(G, items));
  int grid = 0;
  void* args[] = {&k, &c, &p, (void*)&S, &lds, (void*)&P, &ldp, &l, &X, &ldx, &T, &ldt};
#define RB_RI(V)                                                                                           \
  if (p <= V) return coop_launch(richardson_v3<V>, sizeof(RichSmem<V>), args, st, G3, &grid, "rb_ls_richardson");
  RB_RI(8) RB_RI(16) RB_RI(24) RB_RI(32) RB_RI(40) RB_RI(48) RB_RI(64)
#undef RB_RI
  return RB_EINVAL;
}

int sketched_cholqr_small(int k, int p, const double* Sp, int64_t lds, double* R, int64_t ldr, double* Sout,
                          int64_t ldso, int* info, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(k >= 1 && p >= 1 && p <= 64 && Sp && R && Sout && info && lds >= k && ldr >= p && ldso >= k,
             "rb_sketched_cholqr_small: bad args (k=%d p=%d)", k, p);
  // CTAs: row slices of <= 64 rows for the Gram (one load round each), at
  // least one row per thread for the solve
  const int G = std::max(1, std::min(sm_count(), std::max((k + 63) / 64, (k + 255) / 256)));
  int ks = (k + G - 1) / G;
  const size_t need = ((size_t)G * p * p + 2 * (size_t)p * p + p) * sizeof(double);
  RB_REQUIRE(ws && wsb >= need, "rb_sketched_cholqr_small: workspace too small");
  int grid = 0;
  void* args[] = {&k, &p, (void*)&Sp, &lds, &R, &ldr, &Sout, &ldso, &info, &ws, &ks};
  const size_t sm = std::max((size_t)ks * p, (size_t)(2 * p * p + p)) * sizeof(double);
#define RB_CQ(V)                                                                                            \
  if (p <= V) return coop_launch(cholqr_v4<V>, sm, args, st, G, &grid, "rb_sketched_cholqr_small");
  RB_CQ(8) RB_CQ(16) RB_CQ(24) RB_CQ(32) RB_CQ(40) RB_CQ(48) RB_CQ(64)
#undef RB_CQ
  return RB_EINVAL;
}

int certify(int k, int m, const double* S, int64_t lds, const double* P, int64_t ldp, const double* R, int64_t ldr,
            double* out, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(k >= 1 && m >= 1 && S && P && R && out && lds >= k && ldp >= k && ldr >= m,
             "rb_certify: bad args (k=%d m=%d)", k, m);
  const int max_grid = sm_count();
  const int mt = (m + kTM - 1) / kTM, kt = (k + kTM - 1) / kTM;
  const size_t need = ((size_t)(mt * mt + kt * mt) + 2 * (size_t)max_grid) * kTM * 64 * sizeof(double) +
                      3 * (size_t)max_grid * sizeof(double);
  RB_REQUIRE(ws && wsb >= need, "rb_certify: workspace too small (%zu < %zu)", wsb, need);
  int grid = 0;
  void* args[] = {&k, &m, (void*)&S, &lds, (void*)&P, &ldp, (void*)&R, &ldr, &out, &ws};
  return coop_launch(certify_coop, tile_smem<64>(), args, st, max_grid, &grid, "rb_certify");
}

// l2_plus_cholqr without a host branch (rbgs.py:293-302): both outcomes of
// the Gram stage are computed on the device -- (A) R' = chol(Q'^T Q') then
// the sketched CholQR of Q' R'^{-1}, (B) the one-pass sketched CholQR of Q'
// (the same R_ii in exact arithmetic, used when Q'^T Q' is numerically
// indefinite) -- and this kernel keeps A when info[0] == 0, else B, writing
// the chosen R_ii, S_i and status word (info[1] = the chosen path's
// Cholesky info; info[0] is only the selector).
__global__ void l2_select_kernel(int k, int p, const int* __restrict__ info_sel, const int* __restrict__ info_a,
                                 const int* __restrict__ info_b, const double* __restrict__ Ra, int64_t ldra,
                                 const double* __restrict__ Sa, int64_t ldsa, const double* __restrict__ Rb,
                                 int64_t ldrb, const double* __restrict__ Sb, int64_t ldsb, double* __restrict__ R,
                                 int64_t ldr, double* __restrict__ S, int64_t lds, int* __restrict__ info_out) {
  const bool a = *info_sel == 0;
  const int64_t tot = (int64_t)k * p + (int64_t)p * p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < (int64_t)k * p) {
      const int r = (int)(e % k), j = (int)(e / k);
      S[r + j * lds] = a ? Sa[r + j * ldsa] : Sb[r + j * ldsb];
    } else {
      const int64_t f = e - (int64_t)k * p;
      const int i = (int)(f % p), j = (int)(f / p);
      R[i + j * ldr] = a ? Ra[i + j * ldra] : Rb[i + j * ldrb];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *info_out = a ? *info_a : *info_b;
}

int l2_select(int k, int p, const int* info_sel, const int* info_a, const int* info_b, const double* Ra, int64_t ldra,
              const double* Sa, int64_t ldsa, const double* Rb, int64_t ldrb, const double* Sb, int64_t ldsb, double* R,
              int64_t ldr, double* S, int64_t lds, int* info_out, cudaStream_t st) {
  RB_REQUIRE(k >= 1 && p >= 1 && info_sel && info_a && info_b && Ra && Sa && Rb && Sb && R && S && info_out,
             "rb_l2_select: bad args");
  const int64_t tot = (int64_t)k * p + (int64_t)p * p;
  RB_KLAUNCH l2_select_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 2 * sm_count()), 256, 0, st>>>(
      k, p, info_sel, info_a, info_b, Ra, ldra, Sa, ldsa, Rb, ldrb, Sb, ldsb, R, ldr, S, lds, info_out);
  return check_launch("rb_l2_select");
}

int gemm_f64(int tA, int tB, int m, int n, int k, double alpha, const double* A, int64_t lda, const double* B,
             int64_t ldb, double beta, double* C, int64_t ldc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(m >= 0 && n >= 0 && k >= 0 && C && ldc >= std::max(m, 1) && tB == 0 &&
                 (k == 0 || (A && B && lda >= (tA ? k : m) && ldb >= k)),
             "rb_gemm_f64: bad args (op(B) must be B)");
  return gemm_generic<double>(tA, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, wsb, st, "rb_gemm_f64");
}

int gemm_f32(int tA, int tB, int m, int n, int k, float alpha, const float* A, int64_t lda, const float* B,
             int64_t ldb, float beta, float* C, int64_t ldc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(m >= 0 && n >= 0 && k >= 0 && C && ldc >= std::max(m, 1) && tB == 0 &&
                 (k == 0 || (A && B && lda >= (tA ? k : m) && ldb >= k)),
             "rb_gemm_f32: bad args (op(B) must be B)");
  return gemm_generic<float>(tA, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, ws, wsb, st, "rb_gemm_f32");
}

// Upper triangle of C = alpha A^T A + beta C (the full product is formed;
// the strictly lower part of C is written too)
int syrk_f64(int n, int64_t k, double alpha, const double* A, int64_t lda, double beta, double* C, int64_t ldc,
             void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(n >= 0 && k >= 0 && C && ldc >= std::max(n, 1) && (k == 0 || (A && lda >= k)), "rb_syrk_f64: bad args");
  // alpha = 1, beta in {0, 1} (the GMRES basis Gram): 64-column blocks on
  // the FP64 tensor pipe (rb_cross: mma.sync m16n8k4 f64), upper block pairs
  // only -- the strictly lower blocks of C are left untouched.  Each pair
  // re-reads its two column slabs (10 pairs at n = 244: 170 GB at the C4
  // size, 27 ms of HBM time against 134 ms for the CUDA-core tile kernel).
  static const int blk = getenv("RB_SYRK_BLOCKS") ? atoi(getenv("RB_SYRK_BLOCKS")) : 1;
  if (blk && alpha == 1.0 && (beta == 0.0 || beta == 1.0) && k > 0 && n > 0) {
    for (int bi = 0; bi < n; bi += 64) {
      const int wi = std::min(64, n - bi);
      for (int bj = bi; bj < n; bj += 64) {
        const int wj = std::min(64, n - bj);
        const int rc = cross(RB_F64, RB_F64, k, wi, wj, A + (int64_t)bi * lda, lda, A + (int64_t)bj * lda, lda,
                             C + bi + (int64_t)bj * ldc, ldc, beta == 1.0 ? 1 : 0, ws, wsb, st);
        if (rc != RB_OK) return rc;
      }
    }
    return RB_OK;
  }
  // tiles entirely below the diagonal are skipped (C's strictly lower tiles
  // are left untouched): 6 of 8 tiles at n = 244
  return gemm_generic<double>(1, n, n, k, alpha, A, lda, A, lda, beta, C, ldc, ws, wsb, st, "rb_syrk_f64", 1);
}

}  // namespace rb
