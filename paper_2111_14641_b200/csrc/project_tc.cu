// Step 3 on the tensor pipe (RB_ORDER_TC): Qp = fl32(W - Q X) with Q X
// formed by tcgen05.mma kind::tf32 as three products of the split operands
//   Q = Qh + Ql,  X = Xh + Xl   (Qh = rna_tf32(Q), Ql = Q - Qh exactly in
//   binary32, then rounded to tf32 by the MMA; the same for fl32(X))
//   Q X ~= Qh Xh + Qh Xl + Ql Xh  (fp32 accumulation in TMEM)
// -- "3xTF32", about binary32 accuracy (error ~2^-21 of |Q||X| per product
// plus fp32 accumulation), NOT the reference's rounding order
// (kernels.py:171-209 rounds every product and difference separately).  It
// is the fast order of SURVEY.md 8(d) ("HBM if on tensor cores") for inputs
// whose R is insensitive to the Step-3 rounding order: bench.py measures the
// oracle drift per config and uses it only where that drift is <= 1e-6
// (C5's column-scaled family: tests/test_gpu_scale.py); the trig family
// (C1/C2) keeps the bit-exact reference order.
//
// Persistent CTAs, 12 warps:
//   warp 0  producer: per (row tile, 32-column chunk of Q) 32 bulk copies of
//           the chunk's Q column segments (128 rows x 4 B each) and one of
//           the pre-split X planes (prep_x_tf32), onto a transaction mbarrier
//   warp 1  MMA issuer: 4 k-steps x 3 MMAs (M = 128, N = NP, K = 8) per chunk
//   warps 4-7  converters: raw Q chunk -> Qh, Ql in the UMMA K-major
//           no-swizzle layout ([k/4][row][16 B]), one row per thread
//   warps 8-11 epilogue: TMEM -> registers (double-buffered accumulator),
//           Qp = W - D, the norm partials of rbgs.py:373-374
// Algorithmic bytes per call: 4 n (c + 2 p) (Q, W read; Qp written).
//
// v2 (default; RB_TC_V=1 selects the first kernel above): Q tiles arrive by
// 2-D TMA tensor copies (128-byte swizzle) straight in the UMMA MN-major
// operand layout -- a column-major Q tile IS MN-major, so nothing is
// transposed -- the converters only split each entry in place (hi = rna_tf32,
// lo = rna_tf32(q - hi), an elementwise pass that is layout-agnostic), one X
// chunk serves FOUR 128-row tiles (TMEM: 2 x 4 accumulators), the raw ring
// is 6 stages deep (96 KB in flight per SM) and the epilogue prefetches its
// W row into registers before the accumulators are ready.
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "tc.cuh"

namespace rb {

int sm_count();

namespace {

constexpr int kTM = 128;      // rows per tile (UMMA M)
constexpr int kKC = 32;       // Q columns (K) per chunk
constexpr int kTcThreads = 384;
constexpr int kStages = 3;

template <int NP>
struct TcSmem {
  float raw[kStages][kKC][kTM];                 // Q chunk as loaded: [k][row]
  uint8_t ah[kStages][kKC / 4][kTM][16];        // Qh, K-major core matrices
  uint8_t al[kStages][kKC / 4][kTM][16];        // Ql
  uint8_t bx[kStages][2][kKC / 4][NP][16];      // Xh, Xl: [plane][k/4][n][16 B]
  uint64_t full[kStages], conv[kStages], empty[kStages];
  uint64_t tfull[2], tempty[2];
  uint32_t tbase;
  double red[4][2];
};

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  // D = F32 (bits 4-5 = 1), A = B = TF32 (2), both K-major, N >> 3, M >> 4
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Xs (global, per chunk ch: [plane][k/4][n][16 B], NP columns, zero padded
// beyond c rows and p columns): the binary32 rounding of X (the reference's
// cast, kernels.py:192) split into tf32 hi and lo parts.
__global__ void prep_x_tf32(int c, int p, int NP, int nch, const double* __restrict__ X, int64_t ldx,
                            float* __restrict__ Xs, int stacked) {
  const int64_t tot = (int64_t)nch * kKC * NP;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int n = (int)(e % NP);
    const int64_t kk = e / NP;  // global k
    const int ch = (int)(kk / kKC), k = (int)(kk % kKC);
    float hi = 0.f, lo = 0.f;
    if (kk < c && n < p) {
      const float x = __double2float_rn(X[kk + (int64_t)n * ldx]);
      hi = rna_tf32(x);
      lo = x - hi;  // exact
    }
    // float index inside the chunk block: plane, k/4, n, k%4
    const int64_t base = (int64_t)ch * 2 * (kKC / 4) * NP * 4;
    if (stacked) {  // v2: [k/4][Xh rows | Xl rows][16 B]
      Xs[base + ((int64_t)(k / 4) * 2 * NP + n) * 4 + (k & 3)] = hi;
      Xs[base + ((int64_t)(k / 4) * 2 * NP + NP + n) * 4 + (k & 3)] = lo;
    } else {
      Xs[base + ((int64_t)(0 * (kKC / 4) + k / 4) * NP + n) * 4 + (k & 3)] = hi;
      Xs[base + ((int64_t)(1 * (kKC / 4) + k / 4) * NP + n) * 4 + (k & 3)] = lo;
    }
  }
}

template <int NP, typename TW>
__global__ void __launch_bounds__(kTcThreads, 1)
project_tc(int64_t n, int c, int p, const float* __restrict__ Q, int64_t ldq, const float* __restrict__ Xs,
           const TW* W, int64_t ldw, float* Qp, int64_t ldqp, double* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TcSmem<NP>& S = *reinterpret_cast<TcSmem<NP>*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ntiles = n / kTM;  // the caller handles the ragged tail rows
  const int nch = (c + kKC - 1) / kKC;
  // this CTA's tiles: blockIdx.x, blockIdx.x + gridDim.x, ...
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t steps = my_tiles * nch;
  constexpr uint32_t kBBytes = 2 * (kKC / 4) * NP * 16;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.conv[s], 128);
      tc::mbar_init(&S.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], 128);
    }
    tc::mbar_fence_init();
  }
  if (warp == 2) tc::tmem_alloc(&S.tbase, 128);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = S.tbase;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      for (int64_t g = 0; g < steps; ++g) {
        const int s = (int)(g % kStages);
        if (g >= kStages) tc::mbar_wait(&S.empty[s], (uint32_t)((g / kStages) - 1) & 1u);
        const int64_t tile = blockIdx.x + (g / nch) * gridDim.x;
        const int ch = (int)(g % nch);
        const int l0 = ch * kKC, lc = min(kKC, c - l0);
        tc::mbar_arrive_expect_tx(&S.full[s], (uint32_t)(lc * kTM * 4) + kBBytes);
        const float* src = Q + tile * kTM + (int64_t)l0 * ldq;
        for (int u = 0; u < lc; ++u) tc::bulk_g2s(&S.raw[s][u][0], src + (int64_t)u * ldq, kTM * 4, &S.full[s]);
        tc::bulk_g2s(&S.bx[s][0][0][0][0], Xs + (int64_t)ch * (kBBytes / 4), kBBytes, &S.full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t ID = idesc_tf32(kTM, NP);
      for (int64_t g = 0; g < steps; ++g) {
        const int s = (int)(g % kStages);
        const int64_t it = g / nch;  // tile iteration of this CTA
        const int ch = (int)(g % nch);
        const int buf = (int)(it & 1);
        // (the first use of each accumulator buffer needs no hand-back)
        if (ch == 0 && it >= 2) tc::mbar_wait(&S.tempty[buf], (uint32_t)(((it >> 1) - 1) & 1));
        tc::mbar_wait(&S.conv[s], (uint32_t)((g / kStages) & 1));
        tc::tc_fence_after();
        const uint32_t d = tbase + buf * 64;
#pragma unroll
        for (int ks = 0; ks < kKC / 8; ++ks) {
          // K = 8 tf32 = 32 bytes = two 16-byte core-matrix columns (LBO apart)
          const uint64_t ah = tc::sdesc_kmajor(tc::smem_u32(&S.ah[s][2 * ks][0][0]), kTM * 16, 128);
          const uint64_t al = tc::sdesc_kmajor(tc::smem_u32(&S.al[s][2 * ks][0][0]), kTM * 16, 128);
          const uint64_t bh = tc::sdesc_kmajor(tc::smem_u32(&S.bx[s][0][2 * ks][0][0]), NP * 16, 128);
          const uint64_t bl = tc::sdesc_kmajor(tc::smem_u32(&S.bx[s][1][2 * ks][0][0]), NP * 16, 128);
          const uint32_t first = (ch == 0 && ks == 0) ? 0u : 1u;
          mma_tf32(d, ah, bh, ID, first);
          mma_tf32(d, ah, bl, ID, 1u);
          mma_tf32(d, al, bh, ID, 1u);
        }
        tc::mma_commit(&S.empty[s]);
        if (ch == nch - 1) tc::mma_commit(&S.tfull[buf]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- converters: one row per thread ----------------
    const int r = tid - 128;
    for (int64_t g = 0; g < steps; ++g) {
      const int s = (int)(g % kStages);
      const int ch = (int)(g % nch);
      const int lc = min(kKC, c - ch * kKC);
      tc::mbar_wait(&S.full[s], (uint32_t)((g / kStages) & 1));
#pragma unroll
      for (int kc = 0; kc < kKC / 4; ++kc) {
        float4 h, l;
        float* hp = &h.x;
        float* lp = &l.x;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = 4 * kc + t;
          const float q = k < lc ? S.raw[s][k][r] : 0.f;
          const float qh = rna_tf32(q);
          hp[t] = qh;
          lp[t] = q - qh;  // exact
        }
        *reinterpret_cast<float4*>(&S.ah[s][kc][r][0]) = h;
        *reinterpret_cast<float4*>(&S.al[s][kc][r][0]) = l;
      }
      tc::fence_proxy_async_smem();  // generic-proxy stores -> tensor-core reads
      tc::mbar_arrive(&S.conv[s]);
    }
  } else if (warp >= 8) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quadrant
    const int rr = q * 32 + lane;
    double w2 = 0.0, q2 = 0.0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int buf = (int)(it & 1);
      const int64_t row = (blockIdx.x + it * gridDim.x) * kTM + rr;
      tc::mbar_wait(&S.tfull[buf], (uint32_t)((it >> 1) & 1));
      tc::tc_fence_after();
      const uint32_t la = tbase + buf * 64 + ((uint32_t)(q * 32) << 16);
#pragma unroll
      for (int j0 = 0; j0 < NP; j0 += 8) {
        uint32_t v[8];
        tc::tmem_ld8(la + j0, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int j = j0 + jj;
          if (j < p) {
            const TW wv = W[row + (int64_t)j * ldw];
            w2 += (double)wv * (double)wv;
            const float out = __fsub_rn((float)wv, __uint_as_float(v[jj]));
            Qp[row + (int64_t)j * ldqp] = out;
            q2 += (double)out * (double)out;
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[buf]);
    }
    // CTA partial of the two norms (fixed order: warps 8..11, then lanes)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      w2 += __shfl_xor_sync(0xffffffffu, w2, o);
      q2 += __shfl_xor_sync(0xffffffffu, q2, o);
    }
    if (lane == 0) {
      S.red[q][0] = w2;
      S.red[q][1] = q2;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (partial && tid == 256) {
      double a = 0.0, b = 0.0;
      for (int i = 0; i < 4; ++i) {
        a += S.red[i][0];
        b += S.red[i][1];
      }
      partial[2 * blockIdx.x] = a;
      partial[2 * blockIdx.x + 1] = b;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tbase, 128);
}


// ===================================================================== v2
constexpr int kRA = 8;   // raw / hi stages (TMA ring)
constexpr int kRL = 2;   // lo stages
constexpr int kRX = 2;   // X-plane stages
// 128-row tiles per super-tile (they share one X chunk).  Each tile owns TWO
// accumulators of NP columns: D1 = Qh Xh and D2 = Qh Xl + Ql Xh.  The tensor
// pipe truncates its binary32 accumulator at every MMA (measured: the error
// grows with the number of accumulating MMAs, not with 2^-22), so the small
// terms are kept out of the large accumulator and added once, in binary32
// round-to-nearest, by the epilogue.  TMEM: 2 buffers x kSub x 2 NP <= 512.
__host__ __device__ constexpr int sub_tiles(int NP) { return NP <= 32 ? 4 : 2; }

template <int NP>
struct Tc2Smem {
  // one stage: 4 row blocks of 32 rows, each [k = 32][32 floats] (128-B rows,
  // 32-B chunks swizzled with k mod 4): LBO = 4 KB between row blocks,
  // SBO = 512 B between 4-k groups, 1 KB per K = 8 MMA step
  float raw[kRA][4][kKC][32];
  float lo[kRL][4][kKC][32];
  uint8_t bx[kRX][kKC / 4][2 * NP][16];  // [Xh | Xl] stacked along N: K-major core matrices
  uint64_t full[kRA], done[kRA], conv[kRL], xfull[kRX], xempty[kRX];
  uint64_t tfull[2], tempty[2];
  uint32_t tbase;
  double red[4][2];
};

// MN-major operand of 32-bit elements.  Measured on B200 (tools/tc_probe.py
// map): with a_major = MN, kind::tf32 accepts ONLY the layout type
// SWIZZLE_128B_BASE32B (1) -- types 0 / 2 / 4 / 6 make the MMA a silent
// no-op -- i.e. 128-byte rows of 32 consecutive M entries, 32-byte chunks
// XOR-swizzled with the row index mod 4 (cute: Swizzle<2,5,2>), which is
// what a TMA tensor copy with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B writes.
// LBO = byte distance between 32-row M blocks, SBO = between 4-row K groups.
__device__ __forceinline__ uint64_t sdesc_mn_b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;  // version (sm_100)
  d |= (uint64_t)1u << 61;  // SWIZZLE_128B_BASE32B
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32_amn(int M, int N) {
  return idesc_tf32(M, N) | (1u << 15);  // A MN-major, B K-major
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* tmap, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(tc::smem_u32(smem_dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(tc::smem_u32(bar))
      : "memory");
}

constexpr int kTc2Threads = 512;  // 4 role warps + 8 converter warps + 4 epilogue warps
constexpr int kConvThreads = 256;

template <int NP, typename TW>
__global__ void __launch_bounds__(kTc2Threads, 1)
project_tc2(const __grid_constant__ CUtensorMap tmq, int64_t n, int c, int p, const float* __restrict__ Xs,
            const TW* W, int64_t ldw, float* Qp, int64_t ldqp, double* __restrict__ partial) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Tc2Smem<NP>& S = *reinterpret_cast<Tc2Smem<NP>*>(
      (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kSub = sub_tiles(NP);
  const int64_t ntiles = n / kTM;
  const int64_t nsuper = (ntiles + kSub - 1) / kSub;
  const int nch = (c + kKC - 1) / kKC;
  const int64_t my_super = nsuper > blockIdx.x ? (nsuper - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  constexpr uint32_t kBBytes = 2 * (kKC / 4) * NP * 16;
  constexpr uint32_t kABytes = kTM * kKC * 4;
  constexpr uint32_t kAccCols = kSub * 2 * NP;                 // one accumulator buffer: [D1 | D2] per tile
  constexpr uint32_t kAlloc = 2 * kAccCols <= 128 ? 128 : 2 * kAccCols <= 256 ? 256 : 512;
  static_assert(2 * kAccCols <= 512, "TMEM");

  if (tid == 0) {
    for (int s = 0; s < kRA; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.done[s], 1);
    }
    for (int s = 0; s < kRL; ++s) tc::mbar_init(&S.conv[s], kConvThreads);
    for (int s = 0; s < kRX; ++s) {
      tc::mbar_init(&S.xfull[s], 1);
      tc::mbar_init(&S.xempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&S.tfull[b], 1);
      tc::mbar_init(&S.tempty[b], 128);
    }
    tc::mbar_fence_init();
  }
  if (warp == 2) tc::tmem_alloc(&S.tbase, kAlloc);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = S.tbase;
  // sub-tiles of super-tile number `it` of this CTA
  auto nsub_of = [&](int64_t it) -> int {
    const int64_t t0 = (blockIdx.x + it * gridDim.x) * kSub;
    return (int)min((int64_t)kSub, ntiles - t0);
  };

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int64_t g = 0, gx = 0;
      for (int64_t it = 0; it < my_super; ++it) {
        const int64_t row0 = (blockIdx.x + it * gridDim.x) * kSub * kTM;
        const int nsub = nsub_of(it);
        for (int ch = 0; ch < nch; ++ch, ++gx) {
          const int xs = (int)(gx % kRX);
          if (gx >= kRX) tc::mbar_wait(&S.xempty[xs], (uint32_t)((gx / kRX) - 1) & 1u);
          tc::mbar_arrive_expect_tx(&S.xfull[xs], kBBytes);
          tc::bulk_g2s(&S.bx[xs][0][0][0], Xs + (int64_t)ch * (kBBytes / 4), kBBytes, &S.xfull[xs]);
          for (int t = 0; t < nsub; ++t, ++g) {
            const int s = (int)(g % kRA);
            if (g >= kRA) tc::mbar_wait(&S.done[s], (uint32_t)((g / kRA) - 1) & 1u);
            tc::mbar_arrive_expect_tx(&S.full[s], kABytes);
            const int r = (int)(row0 + (int64_t)t * kTM);
#pragma unroll
            for (int b = 0; b < 4; ++b) tma_load_2d(&S.raw[s][b][0][0], &tmq, r + 32 * b, ch * kKC, &S.full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t ID1 = idesc_tf32_amn(kTM, NP), ID2 = idesc_tf32_amn(kTM, 2 * NP);
      int64_t g = 0, gx = 0;
      for (int64_t it = 0; it < my_super; ++it) {
        const int buf = (int)(it & 1);
        const int nsub = nsub_of(it);
        if (it >= 2) tc::mbar_wait(&S.tempty[buf], (uint32_t)(((it >> 1) - 1) & 1));
        for (int ch = 0; ch < nch; ++ch, ++gx) {
          const int xs = (int)(gx % kRX);
          tc::mbar_wait(&S.xfull[xs], (uint32_t)((gx / kRX) & 1));
          for (int t = 0; t < nsub; ++t, ++g) {
            const int s = (int)(g % kRA), sl = (int)(g % kRL);
            tc::mbar_wait(&S.conv[sl], (uint32_t)((g / kRL) & 1));
            tc::tc_fence_after();
            const uint32_t d = tbase + buf * kAccCols + t * 2 * NP;
#pragma unroll
            for (int ks = 0; ks < kKC / 8; ++ks) {
              const uint64_t ah = sdesc_mn_b32(tc::smem_u32(&S.raw[s][0][8 * ks][0]), kKC * 128, 512);
              const uint64_t al = sdesc_mn_b32(tc::smem_u32(&S.lo[sl][0][8 * ks][0]), kKC * 128, 512);
              const uint64_t bb = tc::sdesc_kmajor(tc::smem_u32(&S.bx[xs][2 * ks][0][0]), 2 * NP * 16, 128);
              const uint32_t acc = (ch == 0 && ks == 0) ? 0u : 1u;
              mma_tf32(d, ah, bb, ID2, acc);       // [D1 | D2] (+)= Qh [Xh | Xl]
              mma_tf32(d + NP, al, bb, ID1, 1u);  // D2 += Ql Xh
            }
            tc::mma_commit(&S.done[s]);
          }
          tc::mma_commit(&S.xempty[xs]);
        }
        tc::mma_commit(&S.tfull[buf]);
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // ---------------- converters: elementwise split ----------------
    const int t128 = tid - 128;  // 0 .. kConvThreads - 1
    int64_t total = 0;
    for (int64_t it = 0; it < my_super; ++it) total += (int64_t)nsub_of(it) * nch;
    for (int64_t g = 0; g < total; ++g) {
      const int s = (int)(g % kRA), sl = (int)(g % kRL);
      tc::mbar_wait(&S.full[s], (uint32_t)((g / kRA) & 1));
      // lo[sl] was last read by the MMAs of stage g - kRL
      if (g >= kRL) tc::mbar_wait(&S.done[(int)((g - kRL) % kRA)], (uint32_t)(((g - kRL) / kRA) & 1));
      const float4* src = reinterpret_cast<const float4*>(&S.raw[s][0][0][0]);
      float4* dlo = reinterpret_cast<float4*>(&S.lo[sl][0][0][0]);
#pragma unroll
      for (int i = 0; i < (int)(kABytes / 16 / kConvThreads); ++i) {
        // hi = the entry truncated to tf32 -- what the tensor pipe reads from
        // the raw binary32 word (it ignores the low 13 bits), so the raw
        // stage is used as it arrived; lo = rna_tf32(q - hi), q - hi exact
        const float4 v = src[i * kConvThreads + t128];
        float4 l;
        l.x = rna_tf32(v.x - __uint_as_float(__float_as_uint(v.x) & 0xffffe000u));
        l.y = rna_tf32(v.y - __uint_as_float(__float_as_uint(v.y) & 0xffffe000u));
        l.z = rna_tf32(v.z - __uint_as_float(__float_as_uint(v.z) & 0xffffe000u));
        l.w = rna_tf32(v.w - __uint_as_float(__float_as_uint(v.w) & 0xffffe000u));
        dlo[i * kConvThreads + t128] = l;
      }
      tc::fence_proxy_async_smem();  // generic-proxy stores -> tensor-core reads
      tc::mbar_arrive(&S.conv[sl]);
    }
  } else if (warp >= 12) {
    // ---------------- epilogue: one row per thread ----------------
    const int q = warp & 3;
    const int rr = q * 32 + lane;
    double w2 = 0.0, q2 = 0.0;
    for (int64_t it = 0; it < my_super; ++it) {
      const int buf = (int)(it & 1);
      const int nsub = nsub_of(it);
      const int64_t row0 = (blockIdx.x + it * gridDim.x) * kSub * kTM;
      for (int t = 0; t < nsub; ++t) {
        const int64_t row = row0 + (int64_t)t * kTM + rr;
        // this row of W into registers while the accumulators are busy, in
        // column groups of <= 32 (512 threads: 128 registers per thread)
        constexpr int kCG = NP < 32 ? NP : 32;
        const uint32_t la = tbase + buf * kAccCols + t * 2 * NP + ((uint32_t)(q * 32) << 16);
#pragma unroll
        for (int c0 = 0; c0 < NP; c0 += kCG) {
          TW wv[kCG];
#pragma unroll
          for (int j = 0; j < kCG; ++j)
            wv[j] = (c0 + j < p) ? ld_stream(W + row + (int64_t)(c0 + j) * ldw) : TW(0);
          if (t == 0 && c0 == 0) {
            tc::mbar_wait(&S.tfull[buf], (uint32_t)((it >> 1) & 1));
            tc::tc_fence_after();
          }
#pragma unroll
          for (int j0 = 0; j0 < kCG; j0 += 16) {
            uint32_t v[16], u[16];
            tc::tmem_ld16(la + c0 + j0, v);
            tc::tmem_ld16(la + NP + c0 + j0, u);
            tc::tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int j = c0 + j0 + jj;
              if (j < p) {
                const TW w = wv[j0 + jj];
                w2 += (double)w * (double)w;
                const float dsum = __fadd_rn(__uint_as_float(v[jj]), __uint_as_float(u[jj]));
                const float out = __fsub_rn((float)w, dsum);
                __stcs(Qp + row + (int64_t)j * ldqp, out);
                q2 += (double)out * (double)out;
              }
            }
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[buf]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      w2 += __shfl_xor_sync(0xffffffffu, w2, o);
      q2 += __shfl_xor_sync(0xffffffffu, q2, o);
    }
    if (lane == 0) {
      S.red[q][0] = w2;
      S.red[q][1] = q2;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (partial && tid == 384) {
      double a = 0.0, b = 0.0;
      for (int i = 0; i < 4; ++i) {
        a += S.red[i][0];
        b += S.red[i][1];
      }
      partial[2 * blockIdx.x] = a;
      partial[2 * blockIdx.x + 1] = b;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tbase, kAlloc);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the
// library does not link libcuda: it must load on a box without a driver).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  });
  return fn;
}

int tc_version() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RB_TC_V");
    v = e ? atoi(e) : 2;
  }
  return v;
}

}  // namespace

int project(int, int, int, int, int64_t, int, int, const void*, int64_t, const double*, int64_t, const void*, int64_t,
            void*, int64_t, double*, void*, size_t, cudaStream_t);

// Bytes of workspace project_tc needs: norm pairs per CTA + split X planes.
size_t project_tc_ws_bytes(int c, int p) {
  const int NP = p <= 16 ? 16 : p <= 32 ? 32 : p <= 48 ? 48 : 64;
  const size_t nch = (size_t)(c + kKC - 1) / kKC;
  return ((size_t)sm_count() * 2 * sizeof(double) + 255) / 256 * 256 + nch * 2 * (kKC / 4) * NP * 16 + 256;
}

// Q binary32 (16-B aligned columns), W binary32 or binary64, Qp binary32.
// Rows beyond the last whole 128-row tile go through the CUDA-core FMA order.
int project_tc_launch(int w_dtype, int64_t n, int c, int p, const float* Q, int64_t ldq, const double* X,
                      int64_t ldx, const void* W, int64_t ldw, float* Qp, int64_t ldqp, double* norms2, void* ws,
                      size_t wsb, cudaStream_t st, double* partial_out, int* grid_out) {
  const int NP = p <= 16 ? 16 : p <= 32 ? 32 : p <= 48 ? 48 : 64;
  const int nch = (c + kKC - 1) / kKC;
  const int64_t ntiles = n / kTM;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, sm_count()));
  const size_t part_b = ((size_t)grid * 2 * sizeof(double) + 255) / 256 * 256;
  const size_t xs_b = (size_t)nch * 2 * (kKC / 4) * NP * 16;
  RB_REQUIRE(ws && wsb >= part_b + xs_b && (uintptr_t)ws % 16 == 0, "rb_project (tc): workspace too small");
  double* partial = (double*)ws;
  float* Xs = (float*)((char*)ws + part_b);
  RB_KLAUNCH prep_x_tf32<<<(int)std::min<int64_t>(ceil_div((int64_t)nch * kKC * NP, 256), 4 * sm_count()), 256, 0,
                           st>>>(c, p, NP, nch, X, ldx, Xs, tc_version() >= 2 ? 1 : 0);
  if (tc_version() >= 2 && ntiles > 0) {
    EncodeTiledFn enc = encode_tiled_fn();
    RB_REQUIRE(enc != nullptr, "rb_project (tc): cuTensorMapEncodeTiled unavailable");
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)(ntiles * kTM), (cuuint64_t)c};
    const cuuint64_t strides[1] = {(cuuint64_t)ldq * 4};
    const cuuint32_t box[2] = {32, (cuuint32_t)kKC};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult cr = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)Q, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RB_REQUIRE(cr == CUDA_SUCCESS, "rb_project (tc): cuTensorMapEncodeTiled failed (%d)", (int)cr);
    const int ksub = sub_tiles(NP);
    const int64_t nsuper = (ntiles + ksub - 1) / ksub;
    const int grid2 = (int)std::max<int64_t>(1, std::min<int64_t>(nsuper, sm_count()));
    RB_REQUIRE(grid2 <= grid, "rb_project (tc): partial buffer");
#define RB_TCL2(V, TW)                                                                                       \
  {                                                                                                          \
    const size_t smem = sizeof(Tc2Smem<V>) + 2048;                                                           \
    cudaFuncSetAttribute(project_tc2<V, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    RB_KLAUNCH project_tc2<V, TW><<<grid2, kTc2Threads, smem, st>>>(tm, n, c, p, Xs, (const TW*)W, ldw, Qp,   \
                                                                   ldqp, partial);                        \
  }
    if (w_dtype == RB_F32) {
      if (NP == 16) RB_TCL2(16, float) else if (NP == 32) RB_TCL2(32, float) else if (NP == 48) RB_TCL2(48, float)
      else RB_TCL2(64, float)
    } else {
      if (NP == 16) RB_TCL2(16, double) else if (NP == 32) RB_TCL2(32, double) else if (NP == 48) RB_TCL2(48, double)
      else RB_TCL2(64, double)
    }
#undef RB_TCL2
    *grid_out = grid2;
    (void)partial_out;
    (void)norms2;
    return check_launch("rb_project (tc2)");
  }
#define RB_TCL(V, TW)                                                                                       \
  {                                                                                                         \
    const size_t smem = sizeof(TcSmem<V>) + 1024;                                                           \
    cudaFuncSetAttribute(project_tc<V, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
    RB_KLAUNCH project_tc<V, TW><<<grid, kTcThreads, smem, st>>>(n, c, p, Q, ldq, Xs, (const TW*)W, ldw, Qp, \
                                                                 ldqp, partial);                            \
  }
  if (ntiles > 0) {
    if (w_dtype == RB_F32) {
      if (NP == 16) RB_TCL(16, float) else if (NP == 32) RB_TCL(32, float) else if (NP == 48) RB_TCL(48, float)
      else RB_TCL(64, float)
    } else {
      if (NP == 16) RB_TCL(16, double) else if (NP == 32) RB_TCL(32, double) else if (NP == 48) RB_TCL(48, double)
      else RB_TCL(64, double)
    }
  }
#undef RB_TCL
  *grid_out = ntiles > 0 ? grid : 0;
  (void)partial_out;
  (void)norms2;
  return check_launch("rb_project (tc)");
}

}  // namespace rb
