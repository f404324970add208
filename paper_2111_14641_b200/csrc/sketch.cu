// K1/K2: sketches  out = Theta[:, row0:row0+n] @ X  in fp64
// (rbgs.py:363, :282, :390 -> sketching.py:140-155).
//
//  * dense kinds (gaussian int16 table, rademacher sign bits): split-K
//    register-tiled fp64 GEMM, M = k sketch rows, N = ncols, K = n rows;
//    per-split partials are reduced in a fixed order (deterministic).
//  * srht: pruned subsampled Walsh-Hadamard.  Rows are cut in tiles of
//    T = 2048; with global row i = (g, l), H[s, i] = (-1)^popc(g_s & g) *
//    (-1)^popc(l_s & l), so each tile needs its own 2048-point FWHT and then
//    only a signed gather at the k sampled local indices.  This is the
//    Kronecker split H_n = H_G (x) H_T of SURVEY.md 8(e), with CTAs playing
//    the role of shards.  k <= 1024: one warp per (column, tile), six
//    register stages + one padded smem transpose + five register stages,
//    tiles streamed by per-warp bulk copies (srht_warp); larger k: one CTA
//    per tile, shuffle stages (srht_partial).
//  * sparse_sign: each row i scatters s signed copies of X[i, :] into a
//    shared-memory k x CG accumulator.
#include <type_traits>

#include "common.cuh"
#include "gauss_layout.cuh"
#include "tc.cuh"

namespace rb {

int sm_count();

namespace {

using namespace tc;
constexpr int kThreads = 256;

// ======================= dense (split-K fp64 GEMM) ==========================
constexpr int BM = 128, BK = 16, TM = 8;

// gaussian table: hi (s8, q >> 8) and lo (u8, q & 255) byte planes in the
// tiled layout the tensor-core kernel streams (gauss_layout.cuh).
struct PlaneSrc {
  const uint8_t* t;
  int64_t ld;
  int k;
  __device__ __forceinline__ double at(int r, int64_t i) const {
    return (double)((int)(int8_t)t[gl::q_offset(0, r, i, ld)] * 256 + (int)t[gl::q_offset(1, r, i, ld)]);
  }
};
struct BitSrc {
  const uint32_t* b;
  int64_t ld;  // words per sketch row
  __device__ __forceinline__ double at(int r, int64_t i) const {
    const uint32_t w = b[(int64_t)r * ld + (i >> 5)];
    return ((w >> (i & 31)) & 1u) ? -1.0 : 1.0;
  }
};

template <typename TX, typename Src, int TN>
__global__ void __launch_bounds__(kThreads)
dense_partial(int64_t n, int ncols, const TX* __restrict__ X, int64_t ldx, Src src, int k,
              int64_t chunk, double* __restrict__ ws) {
  // Two shared-memory buffers: the global loads of K step t + 1 are issued
  // into registers before the FMAs of step t and stored to the other buffer
  // after them (one barrier per step) -- at the small all-fp64 shapes (C1)
  // the kernel was bound by exposed load latency, not by the FP64 pipe.
  // Per accumulator the FMA order (kk ascending) is unchanged.
  constexpr int BN = 16 * TN;
  constexpr int kBE = (BN * BK + kThreads - 1) / kThreads;  // B elements per thread
  constexpr bool kPlanes = std::is_same<Src, PlaneSrc>::value;
  constexpr int kAE = kPlanes ? 1 : (BM * BK + kThreads - 1) / kThreads;
  __shared__ __align__(16) double sA[2][BK][BM];
  __shared__ __align__(16) double sB[2][BK][BN];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.x * BM;
  const int64_t kbeg = (int64_t)blockIdx.y * chunk;
  const int64_t kend = min(n, kbeg + chunk);
  double acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = 0.0;

  uint4 hv = make_uint4(0, 0, 0, 0), lv = make_uint4(0, 0, 0, 0);
  double ra[kAE], rb[kBE];
  auto load = [&](int64_t k0) {
    if constexpr (kPlanes) {
      // the gaussian table's 16-row K chunk of a 128-row M tile is one
      // contiguous 2 KB run per plane (gauss_layout.cuh): one 16-byte load
      // of each plane per sketch row
      static_assert(BK == 16 && BM == 128 && kThreads >= BM, "plane tile loader");
      if (threadIdx.x < BM) {
        hv = *reinterpret_cast<const uint4*>(src.t + gl::q_offset(0, m0 + threadIdx.x, k0, src.ld));
        lv = *reinterpret_cast<const uint4*>(src.t + gl::q_offset(1, m0 + threadIdx.x, k0, src.ld));
      }
    } else {
#pragma unroll
      for (int q = 0; q < kAE; ++q) {
        const int e = threadIdx.x + q * kThreads;
        const int r = e / BK, kk = e % BK;
        ra[q] = (e < BM * BK && m0 + r < k && k0 + kk < kend) ? src.at(m0 + r, k0 + kk) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < kBE; ++q) {
      const int e = threadIdx.x + q * kThreads;
      const int j = e / BK, kk = e % BK;
      rb[q] = (e < BN * BK && j < ncols && k0 + kk < kend) ? (double)X[k0 + kk + (int64_t)j * ldx] : 0.0;
    }
  };
  auto store = [&](int buf, int64_t k0) {
    if constexpr (kPlanes) {
      if (threadIdx.x < BM) {
        const int r = threadIdx.x;
        const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          const int hb = (int)(int8_t)((hw[kk >> 2] >> (8 * (kk & 3))) & 255u);
          const int lb = (int)((lw[kk >> 2] >> (8 * (kk & 3))) & 255u);
          sA[buf][kk][r] = (m0 + r < k && k0 + kk < kend) ? (double)(hb * 256 + lb) : 0.0;
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < kAE; ++q) {
        const int e = threadIdx.x + q * kThreads;
        if (e < BM * BK) sA[buf][e % BK][e / BK] = ra[q];
      }
    }
#pragma unroll
    for (int q = 0; q < kBE; ++q) {
      const int e = threadIdx.x + q * kThreads;
      if (e < BN * BK) sB[buf][e % BK][e / BK] = rb[q];
    }
  };

  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0, kbeg);
  }
  __syncthreads();
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int q = 0; q < TM; ++q) a[q] = sA[buf][kk][ty * TM + q];
#pragma unroll
      for (int q = 0; q < TN; ++q) b[q] = sB[buf][kk][tx * TN + q];
#pragma unroll
      for (int q = 0; q < TM; ++q)
#pragma unroll
        for (int t = 0; t < TN; ++t) acc[q][t] = fma(a[q], b[t], acc[q][t]);
    }
    if (more) store(buf ^ 1, k0 + BK);
    __syncthreads();
    buf ^= 1;
  }
  // partial layout: ws[split][j][r] (column-major k x ncols per split)
  double* dst = ws + (int64_t)blockIdx.y * k * ncols;
#pragma unroll
  for (int q = 0; q < TM; ++q) {
    const int r = m0 + ty * TM + q;
#pragma unroll
    for (int t = 0; t < TN; ++t) {
      const int j = tx * TN + t;
      if (r < k && j < ncols) dst[r + (int64_t)j * k] = acc[q][t];
    }
  }
}

// out[r, j] = scale * sum_s ws[s][j][r]  (+ out when accumulate)
__global__ void reduce_splits(const double* __restrict__ ws, int splits, int k, int ncols,
                              double scale, double* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)k * ncols;
  if (e >= tot) return;
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += ws[(int64_t)q * tot + e];
  const int r = (int)(e % k), j = (int)(e / k);
  double* o = out + r + (int64_t)j * ldo;
  *o = accumulate ? *o + scale * s : scale * s;
}

template <typename TX, typename Src>
int dense_sketch(int64_t n, int ncols, const TX* X, int64_t ldx, Src src, int k, double scale,
                 double* out, int64_t ldo, int accumulate, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  const int mt = ceil_div(k, BM);
  const int target = 4 * sm_count();
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (target + mt - 1) / mt));
  const size_t per = (size_t)k * ncols * sizeof(double);
  if ((size_t)splits * per > ws_bytes) splits = (int)std::max<size_t>(1, ws_bytes / per);
  RB_REQUIRE(ws && (size_t)splits * per <= ws_bytes, "sketch: workspace too small");
  int64_t chunk = (n + splits - 1) / splits;
  chunk = (chunk + BK - 1) / BK * BK;
  splits = (int)std::max<int64_t>(1, (n + chunk - 1) / chunk);
  dim3 grid(mt, splits);
  double* w = (double*)ws;
  if (n == 0) {
    splits = 0;
  } else if (ncols <= 16) {
    RB_KLAUNCH dense_partial<TX, Src, 1><<<grid, kThreads, 0, st>>>(n, ncols, X, ldx, src, k, chunk, w);
  } else if (ncols <= 32) {
    RB_KLAUNCH dense_partial<TX, Src, 2><<<grid, kThreads, 0, st>>>(n, ncols, X, ldx, src, k, chunk, w);
  } else if (ncols <= 48) {
    RB_KLAUNCH dense_partial<TX, Src, 3><<<grid, kThreads, 0, st>>>(n, ncols, X, ldx, src, k, chunk, w);
  } else {
    RB_KLAUNCH dense_partial<TX, Src, 4><<<grid, kThreads, 0, st>>>(n, ncols, X, ldx, src, k, chunk, w);
  }
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits<<<ceil_div(tot, 256), 256, 0, st>>>(w, splits, k, ncols, scale, out, ldo, accumulate);
  return check_launch("dense sketch");
}

// ======================= gaussian table fill ================================
__global__ void gaussian_fill_kernel(uint64_t seed, int k, int64_t row0, int64_t nrows,
                                     uint8_t* __restrict__ theta, int64_t ldt, int bits) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;  // quad of sketch rows 4q..4q+3
  if (i >= nrows) return;
  const uint64_t gi = (uint64_t)(row0 + i);
  const u32x4 w = philox4x32_10(u32x4{(uint32_t)gi, (uint32_t)(gi >> 32), (uint32_t)q, kTagGauss},
                                (uint32_t)seed, (uint32_t)(seed >> 32));
  const double sc = 2.3283064365386963e-10;  // 2^-32
  const double ua = ((double)w.x + 0.5) * sc, ub = ((double)w.y + 0.5) * sc;
  const double uc = ((double)w.z + 0.5) * sc, ud = ((double)w.w + 0.5) * sc;
  const double r1 = sqrt(-2.0 * log(ua)), r2 = sqrt(-2.0 * log(uc));
  const double t1 = 6.283185307179586 * ub, t2 = 6.283185307179586 * ud;
  double s1, c1, s2, c2;
  sincos(t1, &s1, &c1);
  sincos(t2, &s2, &c2);
  const double g[4] = {r1 * c1, r1 * s1, r2 * c2, r2 * s2};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int r = 4 * q + t;
    if (r < k) {
      // bits == 8: the same normal on the int8 grid 2^-5, stored as q = 256 q8
      // (hi plane = q8, lo plane = 0: the tensor sketch then skips the lo plane)
      double v = bits == 8 ? 256.0 * fmin(fmax(rint(32.0 * g[t]), -127.0), 127.0)
                           : fmin(fmax(rint(2048.0 * g[t]), -32767.0), 32767.0);
      const int q = (int)v;
      theta[gl::q_offset(0, r, i, ldt)] = (uint8_t)(q >> 8);   // hi plane (signed byte)
      theta[gl::q_offset(1, r, i, ldt)] = (uint8_t)(q & 255);  // lo plane
    }
  }
}

// ======================= SRHT ==============================================
constexpr int kT = 2048;  // tile rows (2^11)

template <int MS, int CG, typename TX>
__global__ void __launch_bounds__(kThreads)
srht_partial(int64_t n, int ncols, const TX* __restrict__ X, int64_t ldx, int64_t row0,
             const uint32_t* __restrict__ sign_bits, const int64_t* __restrict__ sample, int k,
             int tiles_per_cta, int ntiles, double* __restrict__ ws) {
  __shared__ __align__(16) double z[kT];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.y * CG;
  const int cg = min(CG, ncols - c0);
  // my samples: s = tid + 256 m
  int ls[MS];
  int64_t gs[MS];
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int s = tid + kThreads * m;
    const int64_t idx = s < k ? sample[s] : 0;
    ls[m] = (int)(idx & (kT - 1));
    gs[m] = idx >> 11;
  }
  double acc[MS][CG];
#pragma unroll
  for (int m = 0; m < MS; ++m)
#pragma unroll
    for (int c = 0; c < CG; ++c) acc[m][c] = 0.0;

  const int tbeg = blockIdx.x * tiles_per_cta;
  const int tend = min(ntiles, tbeg + tiles_per_cta);
  const int64_t gtile0 = row0 >> 11;  // global tile of local tile 0
  for (int t = tbeg; t < tend; ++t) {
    const int64_t lbase = (int64_t)t * kT;          // local row of element 0
    const int64_t g = gtile0 + t;                   // global tile index
    const int64_t gbase = (row0 & ~(int64_t)(kT - 1)) + lbase;  // global row of element 0
    // sign bits for my 8 rows: elements e = warp*256 + lane*8 + v
    const int e0 = warp * 256 + lane * 8;
    const uint32_t word = sign_bits[(gbase + e0) >> 5];
    const uint32_t sb = (word >> ((gbase + e0) & 31)) & 0xFFu;
    const int64_t off = (row0 & (kT - 1));  // local row of element e is lbase + e - off
    // per-sample sign of H_G[g_s, g]
    double hs[MS];
#pragma unroll
    for (int m = 0; m < MS; ++m) hs[m] = (__popcll((unsigned long long)(gs[m] & g)) & 1) ? -1.0 : 1.0;
    for (int c = 0; c < cg; ++c) {
      const TX* xc = X + (int64_t)(c0 + c) * ldx;
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int64_t lr = lbase + e0 + q - off;
        double x = (lr >= 0 && lr < n) ? (double)xc[lr] : 0.0;
        v[q] = ((sb >> q) & 1u) ? -x : x;
      }
      // stages on bits 0..2 (in register)
#pragma unroll
      for (int h = 1; h < 8; h <<= 1)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (!(q & h)) {
            const double a = v[q], b = v[q + h];
            v[q] = a + b;
            v[q + h] = a - b;
          }
      // stages on bits 3..7 (lane bits 0..4)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const bool hi = lane & o;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const double pv = __shfl_xor_sync(0xffffffffu, v[q], o);
          v[q] = hi ? pv - v[q] : v[q] + pv;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) z[e0 + q] = v[q];
      __syncthreads();
      // stages on bits 8..10: element j*256 + tid
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = z[q * 256 + tid];
#pragma unroll
      for (int h = 1; h < 8; h <<= 1)
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (!(q & h)) {
            const double a = v[q], b = v[q + h];
            v[q] = a + b;
            v[q + h] = a - b;
          }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 8; ++q) z[q * 256 + tid] = v[q];
      __syncthreads();
#pragma unroll
      for (int m = 0; m < MS; ++m)
        if (tid + kThreads * m < k) acc[m][c] += hs[m] * z[ls[m]];
    }
  }
  // partial layout: ws[blockIdx.x][col][s]
  double* dst = ws + (int64_t)blockIdx.x * k * ncols;
#pragma unroll
  for (int m = 0; m < MS; ++m) {
    const int s = tid + kThreads * m;
    if (s < k)
#pragma unroll
      for (int c = 0; c < CG; ++c)
        if (c < cg) dst[s + (int64_t)(c0 + c) * k] = acc[m][c];
  }
}

// Warp-per-column SRHT (k <= 1024): warp w of the CTA owns column c0 + w for
// every tile of the CTA's range.  Phase A: lane L holds rows e = L + 32 i
// (i < 64, coalesced 128-byte loads) and runs the six stages on bits 5..10
// in registers; a padded per-warp smem transpose (row stride 33, conflict
// free both ways) hands lane L the rows (L + 32 h) * 32 + b (h < 2, b < 32)
// for the five stages on bits 0..4.  The transformed tile goes back to smem
// and each lane gathers its samples s = L + 32 m (accumulators in
// registers).  11 * 2048 / 32 = 704 DADD per lane per tile column: the
// kernel sits at the fp64 add rate ~ the HBM rate of the tile stream.
constexpr int kSW = 8;                 // warps (columns) per CTA

// lane L holds row L of a 32 x 32 bit matrix; returns column L (bit i = row
// i's bit L).  Recursive block swap, one shuffle per level.
__device__ __forceinline__ uint32_t warp_bit_transpose(uint32_t w, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const int j = 16 >> q;
    const uint32_t m = masks[q];
    const uint32_t p = __shfl_xor_sync(0xffffffffu, w, j);
    w = (lane & j) ? ((w & ~m) | ((p & ~m) >> j)) : ((w & m) | ((p & m) << j));
  }
  return w;
}
constexpr int kZS = kT / 32 * 33;      // padded per-warp tile (2112 doubles)

// ST: interior tiles arrive by one bulk copy per (warp, tile) into a per-warp
// staging buffer, issued a tile ahead, so the next tile streams in while the
// current one is transformed (needs 16-B aligned tile starts).
template <int MS, typename TX, bool ST>
__global__ void __launch_bounds__(kSW * 32, 1)
srht_warp(int64_t n, int ncols, const TX* __restrict__ X, int64_t ldx, int64_t row0,
          const uint32_t* __restrict__ sign_bits, const int64_t* __restrict__ sample, int k,
          int tiles_per_cta, int ntiles, double* __restrict__ ws) {
  extern __shared__ __align__(128) double zsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.y * kSW + warp;
  double* zs = zsm + warp * kZS;
  TX* stage = reinterpret_cast<TX*>(zsm + kSW * kZS) + warp * kT;
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<TX*>(zsm + kSW * kZS) + (ST ? kSW * kT : 0)) + warp;
  // sample s: padded smem slot (12 bits) | global tile index << 12, shared by
  // the CTA's warps (kept out of registers)
  uint32_t* stab = reinterpret_cast<uint32_t*>(bar - warp + kSW);
  for (int s = threadIdx.x; s < 32 * MS; s += blockDim.x) {
    const int64_t idx = s < k ? sample[s] : 0;
    const int l = (int)(idx & (kT - 1));
    stab[s] = (uint32_t)((l >> 5) * 33 + (l & 31)) | ((uint32_t)(idx >> 11) << 12);
  }
  __syncthreads();
  if (c >= ncols) return;  // no CTA-wide barriers below
  const TX* xc = X + (int64_t)c * ldx;
  double acc[MS];
#pragma unroll
  for (int m = 0; m < MS; ++m) acc[m] = 0.0;
  const int tbeg = blockIdx.x * tiles_per_cta;
  const int tend = min(ntiles, tbeg + tiles_per_cta);
  const int64_t gtile0 = row0 >> 11;
  const int64_t off = row0 & (kT - 1);
  const int64_t galign = row0 & ~(int64_t)(kT - 1);
  auto interior = [&](int t) {
    const int64_t lb = (int64_t)t * kT - off;
    return lb >= 0 && lb + kT <= n;
  };
  auto prefetch = [&](int t) {  // lane 0 only
    mbar_arrive_expect_tx(bar, kT * sizeof(TX));
    bulk_g2s(stage, xc + ((int64_t)t * kT - off), kT * sizeof(TX), bar);
  };
  uint32_t phase = 0;
  if (ST) {
    if (lane == 0) {
      mbar_init(bar, 1);
      mbar_fence_init();
      if (tbeg < tend && interior(tbeg)) prefetch(tbeg);
    }
    __syncwarp();
  }
  for (int t = tbeg; t < tend; ++t) {
    const int64_t lbase = (int64_t)t * kT - off;  // local row of tile element 0
    const int g = (int)(gtile0 + t);
    const uint32_t* sb = sign_bits + ((galign + (int64_t)t * kT) >> 5);
    double v[64];
    if (ST && interior(t)) {
      mbar_wait(bar, phase);
      phase ^= 1u;
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = (double)stage[lane + 32 * i];
      __syncwarp();
      if (lane == 0 && t + 1 < tend && interior(t + 1)) {
        fence_proxy_async_smem();
        prefetch(t + 1);
      }
    } else if (lbase >= 0 && lbase + kT <= n) {
      // interior tile: 64 unpredicated loads in flight before the first use
      const TX* xt = xc + lbase + lane;
      TX raw[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) raw[i] = __ldg(xt + 32 * i);
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = (double)raw[i];
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const int64_t lr = lbase + lane + 32 * i;
        v[i] = (lr >= 0 && lr < n) ? (double)xc[lr] : 0.0;
      }
      if (ST) {
        __syncwarp();
        if (lane == 0 && t + 1 < tend && interior(t + 1)) prefetch(t + 1);
      }
    }
    // D: lane L needs bit L of sign words i = 0..63 -> transpose the two
    // 32 x 32 bit blocks across the warp (5 shuffle rounds each)
    const uint32_t t0 = warp_bit_transpose(__ldg(sb + lane), lane);
    const uint32_t t1 = warp_bit_transpose(__ldg(sb + 32 + lane), lane);
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      const uint32_t t = i < 32 ? t0 : t1;
      const uint32_t flip = (t << (31 - (i & 31))) & 0x80000000u;
      v[i] = __hiloint2double(__double2hiint(v[i]) ^ (int)flip, __double2loint(v[i]));
    }
#pragma unroll
    for (int h = 1; h < 64; h <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (!(i & h)) {
          const double a = v[i], b = v[i + h];
          v[i] = a + b;
          v[i + h] = a - b;
        }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 64; ++i) zs[i * 33 + lane] = v[i];
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int b = 0; b < 32; ++b) v[h * 32 + b] = zs[(lane + 32 * h) * 33 + b];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1)
#pragma unroll
      for (int i = 0; i < 64; ++i)
        if (!(i & o)) {
          const double a = v[i], b = v[i + o];
          v[i] = a + b;
          v[i + o] = a - b;
        }
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int b = 0; b < 32; ++b) zs[(lane + 32 * h) * 33 + b] = v[h * 32 + b];
    __syncwarp();
#pragma unroll
    for (int m = 0; m < MS; ++m) {
      const uint32_t e = stab[lane + 32 * m];
      const double z = zs[e & 4095u];
      acc[m] += (__popc((e >> 12) & (uint32_t)g) & 1) ? -z : z;
    }
  }
  double* dst = ws + (int64_t)blockIdx.x * k * ncols + (int64_t)c * k;
#pragma unroll
  for (int m = 0; m < MS; ++m)
    if (lane + 32 * m < k) dst[lane + 32 * m] = acc[m];
}

template <typename TX>
int srht_sketch(int64_t n, int ncols, const TX* X, int64_t ldx, int64_t row0, int64_t n_pad,
                const uint32_t* bits, const int64_t* sample, int k, double scale, double* out,
                int64_t ldo, int accumulate, void* ws, size_t ws_bytes, cudaStream_t st) {
  RB_REQUIRE(k <= 8 * kThreads, "srht: k=%d > 2048 unsupported", k);
  RB_REQUIRE(n_pad <= ((int64_t)1 << 31), "srht: n_pad > 2^31 unsupported");
  RB_REQUIRE(n_pad <= kT || (row0 % kT) == 0, "srht: row0 must be a multiple of 2048");
  const int64_t span = (row0 % kT) + n;  // rows covered from the first tile start
  const int ntiles = ceil_div(span, kT);
  const size_t per = (size_t)k * ncols * sizeof(double);
  if (k <= 1024 && !getenv("RB_SRHT_V1")) {
    const int cgroups = ceil_div(ncols, kSW);
    int ctas = std::max(1, std::min(ntiles, sm_count() / cgroups));
    if ((size_t)ctas * per > ws_bytes) ctas = (int)std::max<size_t>(1, ws_bytes / per);
    RB_REQUIRE(ws && (size_t)ctas * per <= ws_bytes, "srht: workspace too small");
    const int tpc = ceil_div(ntiles, ctas);
    ctas = ceil_div(ntiles, tpc);
    const dim3 grid(ctas, cgroups);
    const bool stage = sizeof(TX) == 4 && ((uintptr_t)X % 16) == 0 && ldx % 4 == 0 &&
                       (row0 % kT) % 4 == 0 && !getenv("RB_SRHT_NOSTAGE");
    const size_t smem = (size_t)kSW * kZS * sizeof(double) + (stage ? kSW * kT * sizeof(TX) : 0) + kSW * 8 +
                        (size_t)32 * 32 * sizeof(uint32_t);
    double* w = (double*)ws;
#define RB_SRHTW(M)                                                                                    \
  do {                                                                                                 \
    if (stage) {                                                                                       \
      cudaFuncSetAttribute(srht_warp<M, TX, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      RB_KLAUNCH srht_warp<M, TX, true><<<grid, kSW * 32, smem, st>>>(n, ncols, X, ldx, row0, bits, sample, k, \
                                                                      tpc, ntiles, w);                 \
    } else {                                                                                           \
      cudaFuncSetAttribute(srht_warp<M, TX, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      RB_KLAUNCH srht_warp<M, TX, false><<<grid, kSW * 32, smem, st>>>(n, ncols, X, ldx, row0, bits, sample, \
                                                                       k, tpc, ntiles, w);             \
    }                                                                                                  \
  } while (0)
    if (k <= 64) RB_SRHTW(2);
    else if (k <= 128) RB_SRHTW(4);
    else if (k <= 256) RB_SRHTW(8);
    else if (k <= 512) RB_SRHTW(16);
    else RB_SRHTW(32);
#undef RB_SRHTW
    const int64_t tot = (int64_t)k * ncols;
    RB_KLAUNCH reduce_splits<<<ceil_div(tot, 256), 256, 0, st>>>(w, ctas, k, ncols, scale, out, ldo, accumulate);
    return check_launch("srht sketch");
  }
  const int MS = k <= 256 ? 1 : k <= 512 ? 2 : k <= 1024 ? 4 : 8;
  const int CG = MS >= 8 ? 4 : 8;
  const int cgroups = ceil_div(ncols, CG);
  int ctas = std::max(1, std::min(ntiles, (2 * sm_count() + cgroups - 1) / cgroups));
  if ((size_t)ctas * per > ws_bytes) ctas = (int)std::max<size_t>(1, ws_bytes / per);
  RB_REQUIRE(ws && (size_t)ctas * per <= ws_bytes, "srht: workspace too small");
  const int tpc = ceil_div(ntiles, ctas);
  ctas = ceil_div(ntiles, tpc);
  dim3 grid(ctas, cgroups);
  double* w = (double*)ws;
#define RB_SRHT(M, C) RB_KLAUNCH srht_partial<M, C, TX><<<grid, kThreads, 0, st>>>(n, ncols, X, ldx, row0, bits, sample, k, tpc, ntiles, w)
  if (MS == 1) RB_SRHT(1, 8);
  else if (MS == 2) RB_SRHT(2, 8);
  else if (MS == 4) RB_SRHT(4, 8);
  else RB_SRHT(8, 4);
#undef RB_SRHT
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits<<<ceil_div(tot, 256), 256, 0, st>>>(w, ctas, k, ncols, scale, out, ldo, accumulate);
  return check_launch("srht sketch");
}

// ======================= sparse sign ========================================
// Bucketed accumulation: a CTA streams tiles of kST rows; for every row it
// hashes the s target sketch rows (sparse_sign_column), stages x / sqrt(s)
// in shared memory and counts the targets per sketch row (native 32-bit
// shared atomics); a block scan turns the counts into bucket offsets, the
// (row, sign) entries are scattered into their buckets, and the owner thread
// of each sketch row sums its bucket for all columns of the pass.  This
// replaces s * ncols binary64 shared-memory atomics per row (a CAS loop on
// sm_100) by 2 s integer atomics per row.  Per-CTA partials are reduced in
// CTA order by reduce_splits.
constexpr int kST = 1024;            // rows per tile
constexpr int kSRPT = kST / kThreads;  // rows per thread per tile

template <typename TX, int CG, int SMAX>
__global__ void __launch_bounds__(kThreads)
sparse_bucket_partial(int64_t n, int ncols, const TX* __restrict__ X, int64_t ldx, int64_t row0, uint64_t seed,
                      int k, int s, double* __restrict__ ws) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sx = reinterpret_cast<double*>(smem_raw);          // [kST][CG]
  double* sacc = sx + kST * CG;                               // [k][CG]
  int* cnt = reinterpret_cast<int*>(sacc + (size_t)k * CG);   // [k]
  int* cur = cnt + k;                                         // [k]
  uint32_t* list = reinterpret_cast<uint32_t*>(cur + k);      // [kST * s]
  __shared__ int wsum[kThreads / 32];
  const int c0 = blockIdx.y * CG;
  const int cc = min(CG, ncols - c0);
  const double inv = 1.0 / sqrt((double)s);
  for (int e = threadIdx.x; e < k * CG; e += kThreads) sacc[e] = 0.0;
  const int64_t ntiles = (n + kST - 1) / kST;
  const int per = (k + kThreads - 1) / kThreads;  // scan segment per thread
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t base = tile * kST;
    for (int e = threadIdx.x; e < k; e += kThreads) cnt[e] = 0;
    __syncthreads();
    int tr[kSRPT][SMAX];
    bool live[kSRPT];
#pragma unroll
    for (int u = 0; u < kSRPT; ++u) {
      const int il = threadIdx.x + u * kThreads;
      const int64_t i = base + il;
      live[u] = i < n;
      if (live[u]) {
        sparse_sign_targets<SMAX>((uint64_t)(row0 + i), seed, k, s, tr[u]);
#pragma unroll
        for (int q = 0; q < SMAX; ++q)
          if (q < s) atomicAdd(&cnt[tr[u][q] >> 1], 1);
#pragma unroll
        for (int c = 0; c < CG; ++c) sx[il * CG + c] = c < cc ? (double)X[i + (int64_t)(c0 + c) * ldx] * inv : 0.0;
      }
    }
    __syncthreads();
    // exclusive scan of cnt -> cur (thread t owns bins [t per, (t+1) per))
    int loc = 0;
    for (int j = 0; j < per; ++j) {
      const int r = threadIdx.x * per + j;
      if (r < k) loc += cnt[r];
    }
    int incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += v;
    }
    if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = incl;
    __syncthreads();
    int off = incl - loc;
    for (int w = 0; w < (threadIdx.x >> 5); ++w) off += wsum[w];
    for (int j = 0; j < per; ++j) {
      const int r = threadIdx.x * per + j;
      if (r < k) {
        cur[r] = off;
        off += cnt[r];
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kSRPT; ++u) {
      if (!live[u]) continue;
      const int il = threadIdx.x + u * kThreads;
#pragma unroll
      for (int q = 0; q < SMAX; ++q) {
        if (q < s) {
          const int pos = atomicAdd(&cur[tr[u][q] >> 1], 1);
          list[pos] = ((uint32_t)il << 1) | (uint32_t)(tr[u][q] & 1);
        }
      }
    }
    __syncthreads();
    // owners: cur[r] now holds the END of bucket r
    for (int r = threadIdx.x; r < k; r += kThreads) {
      const int e1 = cur[r], e0 = e1 - cnt[r];
      double acc[CG];
#pragma unroll
      for (int c = 0; c < CG; ++c) acc[c] = sacc[r * CG + c];
      for (int e = e0; e < e1; ++e) {
        const uint32_t v = list[e];
        const double* xr = sx + (v >> 1) * CG;
        if (v & 1u) {
#pragma unroll
          for (int c = 0; c < CG; ++c) acc[c] -= xr[c];
        } else {
#pragma unroll
          for (int c = 0; c < CG; ++c) acc[c] += xr[c];
        }
      }
#pragma unroll
      for (int c = 0; c < CG; ++c) sacc[r * CG + c] = acc[c];
    }
    __syncthreads();
  }
  double* dst = ws + (int64_t)blockIdx.x * k * ncols;
  for (int e = threadIdx.x; e < k * cc; e += kThreads) {
    const int r = e % k, c = e / k;
    dst[r + (int64_t)(c0 + c) * k] = sacc[r * CG + c];
  }
}

template <typename TX, int CG>
size_t sparse_smem(int k, int s) {
  return (size_t)kST * CG * sizeof(double) + (size_t)k * CG * sizeof(double) + 2 * (size_t)k * sizeof(int) +
         (size_t)kST * s * sizeof(uint32_t);
}

// ---- pre-bucketed table (built once per operator shard) --------------------
// Per tile of kST local rows: offs[k + 1] (int32 bucket starts) and the
// tile's s * rows entries (uint16: local row << 1 | negative sign) sorted by
// sketch row, then by local row -- the summation order of every sketch is
// fixed (deterministic) and no hashing or atomics remain on the per-call
// path, which just streams X, the lists and the offsets.
template <int SMAX>
__global__ void __launch_bounds__(kThreads)
sparse_table_build(int64_t nrows, int64_t row0, uint64_t seed, int k, int s, int32_t* __restrict__ offs,
                   uint16_t* __restrict__ lists) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int* cnt = reinterpret_cast<int*>(smem_raw);  // [k]
  int* cur = cnt + k;                           // [k]
  uint16_t* lst = reinterpret_cast<uint16_t*>(cur + k);  // [kST * s]
  __shared__ int wsum[kThreads / 32];
  const int64_t tile = blockIdx.x;
  const int64_t base = tile * kST;
  for (int e = threadIdx.x; e < k; e += kThreads) cnt[e] = 0;
  __syncthreads();
  int tr[kSRPT][SMAX];
  bool live[kSRPT];
#pragma unroll
  for (int u = 0; u < kSRPT; ++u) {
    const int64_t i = base + threadIdx.x + u * kThreads;
    live[u] = i < nrows;
    if (live[u]) {
      sparse_sign_targets<SMAX>((uint64_t)(row0 + i), seed, k, s, tr[u]);
#pragma unroll
      for (int q = 0; q < SMAX; ++q)
        if (q < s) atomicAdd(&cnt[tr[u][q] >> 1], 1);
    }
  }
  __syncthreads();
  const int per = (k + kThreads - 1) / kThreads;
  int loc = 0;
  for (int j = 0; j < per; ++j) {
    const int r = threadIdx.x * per + j;
    if (r < k) loc += cnt[r];
  }
  int incl = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if ((threadIdx.x & 31) >= o) incl += v;
  }
  if ((threadIdx.x & 31) == 31) wsum[threadIdx.x >> 5] = incl;
  __syncthreads();
  int off = incl - loc;
  for (int w = 0; w < (threadIdx.x >> 5); ++w) off += wsum[w];
  int32_t* to = offs + tile * (int64_t)(k + 1);
  for (int j = 0; j < per; ++j) {
    const int r = threadIdx.x * per + j;
    if (r < k) {
      cur[r] = off;
      to[r] = off;
      off += cnt[r];
    }
  }
  if (threadIdx.x == kThreads - 1) to[k] = off;  // last thread's running end = total
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kSRPT; ++u) {
    if (!live[u]) continue;
    const int il = threadIdx.x + u * kThreads;
#pragma unroll
    for (int q = 0; q < SMAX; ++q)
      if (q < s) lst[atomicAdd(&cur[tr[u][q] >> 1], 1)] = (uint16_t)((il << 1) | (tr[u][q] & 1));
  }
  __syncthreads();
  // deterministic order inside each bucket: insertion sort by local row
  for (int r = threadIdx.x; r < k; r += kThreads) {
    const int e1 = cur[r], e0 = e1 - cnt[r];
    for (int a = e0 + 1; a < e1; ++a) {
      const uint16_t v = lst[a];
      int b = a - 1;
      while (b >= e0 && lst[b] > v) {
        lst[b + 1] = lst[b];
        --b;
      }
      lst[b + 1] = v;
    }
  }
  __syncthreads();
  uint16_t* tl = lists + tile * (int64_t)kST * s;
  const int tot = (int)min((int64_t)kST, nrows - base) * s;
  for (int e = threadIdx.x; e < tot; e += kThreads) tl[e] = lst[e];
}

template <typename TX, int CG>
__global__ void __launch_bounds__(kThreads)
sparse_tab_partial(int64_t n, int ncols, const TX* __restrict__ X, int64_t ldx, const int32_t* __restrict__ offs,
                   const uint16_t* __restrict__ lists, int k, int s, double* __restrict__ ws) {
  // x staged column-major (sx[c][il]): random-row reads of one column hit
  // ~distinct banks; the next tile's X, list and offsets are prefetched
  // into registers while the current tile is summed
  constexpr int XPT = kST / kThreads;  // rows per thread per column
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* sx = reinterpret_cast<double*>(smem_raw);          // [CG][kST]
  double* sacc = sx + kST * CG;                               // [k][CG]
  int* so = reinterpret_cast<int*>(sacc + (size_t)k * CG);    // [k + 1]
  uint16_t* sl = reinterpret_cast<uint16_t*>(so + ((k + 1 + 7) & ~7));  // [kST * s], 16-B aligned
  const int c0 = blockIdx.y * CG;
  const int cc = min(CG, ncols - c0);
  const double inv = 1.0 / sqrt((double)s);
  for (int e = threadIdx.x; e < k * CG; e += kThreads) sacc[e] = 0.0;
  const int64_t ntiles = (n + kST - 1) / kST;
  const int LV = (kST * s / 8 + kThreads - 1) / kThreads;  // uint4 of list per thread (<= 8)
  TX px[CG][XPT];  // raw loads: consumed (scaled) only at the smem store
  uint4 pl[8];
  auto fetch = [&](int64_t tile) {
    const int64_t base = tile * kST;
#pragma unroll
    for (int c = 0; c < CG; ++c)
#pragma unroll
      for (int u = 0; u < XPT; ++u) {
        const int64_t i = base + threadIdx.x + u * kThreads;
        px[c][u] = (c < cc && i < n) ? X[i + (int64_t)(c0 + c) * ldx] : TX(0);
      }
    const uint4* tl = reinterpret_cast<const uint4*>(lists + tile * (int64_t)kST * s);
    const int rows = (int)min((int64_t)kST, n - base);
    const int vec = (rows * s + 7) / 8;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < LV) {
        const int e = threadIdx.x + u * kThreads;
        pl[u] = e < vec ? tl[e] : make_uint4(0, 0, 0, 0);
      }
  };
  int64_t tile = blockIdx.x;
  if (tile < ntiles) fetch(tile);
  for (; tile < ntiles; tile += gridDim.x) {
    __syncthreads();  // previous tile consumed
#pragma unroll
    for (int c = 0; c < CG; ++c)
#pragma unroll
      for (int u = 0; u < XPT; ++u) sx[c * kST + threadIdx.x + u * kThreads] = (double)px[c][u] * inv;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < LV && threadIdx.x + u * kThreads < kST * s / 8)
        reinterpret_cast<uint4*>(sl)[threadIdx.x + u * kThreads] = pl[u];
    for (int e = threadIdx.x; e <= k; e += kThreads) so[e] = offs[tile * (int64_t)(k + 1) + e];
    __syncthreads();
    if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);  // in flight during the sums
    for (int r = threadIdx.x; r < k; r += kThreads) {
      const int e0 = so[r], e1 = so[r + 1];
      double acc[CG];
#pragma unroll
      for (int c = 0; c < CG; ++c) acc[c] = sacc[r * CG + c];
      for (int e = e0; e < e1; ++e) {
        const uint32_t v = sl[e];
        const int il = (int)(v >> 1);
        const double sg = (v & 1u) ? -1.0 : 1.0;
#pragma unroll
        for (int c = 0; c < CG; ++c) acc[c] = fma(sg, sx[c * kST + il], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < CG; ++c) sacc[r * CG + c] = acc[c];
    }
  }
  __syncthreads();
  double* dst = ws + (int64_t)blockIdx.x * k * ncols;
  for (int e = threadIdx.x; e < k * cc; e += kThreads) {
    const int r = e % k, c = e / k;
    dst[r + (int64_t)(c0 + c) * k] = sacc[r * CG + c];
  }
}

template <typename TX>
int sparse_sketch_tab(int64_t n, int ncols, const TX* X, int64_t ldx, const int32_t* offs, const uint16_t* lists,
                      int k, int s, double* out, int64_t ldo, int accumulate, void* ws, size_t ws_bytes,
                      cudaStream_t st) {
  constexpr int CG = 4;
  const size_t smem = (size_t)kST * CG * sizeof(double) + (size_t)k * CG * sizeof(double) +
                      (size_t)((k + 1 + 7) & ~7) * sizeof(int) + (size_t)kST * s * sizeof(uint16_t) + 16;
  RB_REQUIRE(smem <= 200 * 1024, "sparse_sign: k too large (%d)", k);
  const int cgroups = ceil_div(ncols, CG);
  const size_t per = (size_t)k * ncols * sizeof(double);
  const int64_t ntiles = (n + kST - 1) / kST;
  int ctas = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (2 * sm_count() + cgroups - 1) / cgroups));
  if ((size_t)ctas * per > ws_bytes) ctas = (int)std::max<size_t>(1, ws_bytes / per);
  RB_REQUIRE(ws && (size_t)ctas * per <= ws_bytes, "sparse_sign: workspace too small");
  cudaFuncSetAttribute(sparse_tab_partial<TX, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (n > 0)
    RB_KLAUNCH sparse_tab_partial<TX, CG><<<dim3(ctas, cgroups), kThreads, smem, st>>>(n, ncols, X, ldx, offs, lists,
                                                                                     k, s, (double*)ws);
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits<<<ceil_div(tot, 256), 256, 0, st>>>((double*)ws, n > 0 ? ctas : 0, k, ncols, 1.0, out, ldo,
                                                    accumulate);
  return check_launch("sparse_sign sketch (table)");
}

template <typename TX>
int sparse_sketch(int64_t n, int ncols, const TX* X, int64_t ldx, int64_t row0, uint64_t seed,
                  int k, int nnz, double* out, int64_t ldo, int accumulate, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  const int s = std::min(nnz, k);
  RB_REQUIRE(s >= 1 && s <= 16, "sparse_sign: nnz must be in [1, 16]");
  constexpr int CG = 4;
  const size_t smem = sparse_smem<TX, CG>(k, s);
  RB_REQUIRE(smem <= 200 * 1024, "sparse_sign: k too large (%d)", k);
  const int cgroups = ceil_div(ncols, CG);
  const size_t per = (size_t)k * ncols * sizeof(double);
  const int64_t ntiles = (n + kST - 1) / kST;
  int ctas = (int)std::max<int64_t>(1, std::min<int64_t>(ntiles, (2 * sm_count() + cgroups - 1) / cgroups));
  if ((size_t)ctas * per > ws_bytes) ctas = (int)std::max<size_t>(1, ws_bytes / per);
  RB_REQUIRE(ws && (size_t)ctas * per <= ws_bytes, "sparse_sign: workspace too small");
#define RB_SB(SM)                                                                                             \
  do {                                                                                                        \
    cudaFuncSetAttribute(sparse_bucket_partial<TX, CG, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                         (int)smem);                                                                          \
    RB_KLAUNCH sparse_bucket_partial<TX, CG, SM><<<dim3(ctas, cgroups), kThreads, smem, st>>>(                \
        n, ncols, X, ldx, row0, seed, k, s, (double*)ws);                                                     \
  } while (0)
  if (n > 0) {
    if (s <= 4) RB_SB(4);
    else if (s <= 8) RB_SB(8);
    else RB_SB(16);
  }
#undef RB_SB
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits<<<ceil_div(tot, 256), 256, 0, st>>>((double*)ws, n > 0 ? ctas : 0, k, ncols, 1.0, out, ldo,
                                                    accumulate);
  return check_launch("sparse_sign sketch");
}

}  // namespace

// ============================== entry points ================================
int gaussian_fill(uint64_t seed, int k, int64_t row0, int64_t nrows, uint8_t* theta, int64_t ldt,
                  cudaStream_t st, int bits) {
  RB_REQUIRE(bits == 16 || bits == 8, "rb_gaussian_fill: bits must be 16 or 8");
  RB_REQUIRE(k >= 1 && k <= 4 * 65535 && nrows >= 0 && ldt >= nrows && ldt % gl::kBK == 0 && theta,
             "rb_gaussian_fill: bad args (ldt must be a multiple of 128)");
  cudaMemsetAsync(theta, 0, (size_t)gl::q_bytes(k, ldt), st);  // zero padding rows / columns
  if (nrows == 0) return check_launch("rb_gaussian_fill");
  dim3 grid(ceil_div(nrows, 256), (k + 3) / 4);
  RB_KLAUNCH gaussian_fill_kernel<<<grid, 256, 0, st>>>(seed, k, row0, nrows, theta, ldt, bits);
  return check_launch("rb_gaussian_fill");
}

// Pre-bucketed sparse-sign table for local rows [0, nrows) of a shard that
// starts at global row row0: offs int32[ntiles][k + 1], lists
// uint16[ntiles][1024 s], ntiles = ceil(nrows / 1024).
int sparse_sign_table(uint64_t seed, int k, int nnz, int64_t row0, int64_t nrows, int32_t* offs, uint16_t* lists,
                      cudaStream_t st) {
  const int s = std::min(nnz, k);
  RB_REQUIRE(s >= 1 && s <= 16 && k >= 1 && k < 32768 && nrows >= 0 && (nrows == 0 || (offs && lists)),
             "rb_sparse_sign_table: bad args");
  const int64_t ntiles = (nrows + kST - 1) / kST;
  const size_t smem = 2 * (size_t)k * sizeof(int) + (size_t)kST * s * sizeof(uint16_t) + 16;
  RB_REQUIRE(smem <= 200 * 1024, "rb_sparse_sign_table: k too large");
  if (ntiles == 0) return check_launch("rb_sparse_sign_table");
#define RB_TB(SM)                                                                                         \
  do {                                                                                                    \
    cudaFuncSetAttribute(sparse_table_build<SM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    RB_KLAUNCH sparse_table_build<SM><<<(unsigned)ntiles, kThreads, smem, st>>>(nrows, row0, seed, k, s, offs, lists); \
  } while (0)
  if (s <= 4) RB_TB(4);
  else if (s <= 8) RB_TB(8);
  else RB_TB(16);
#undef RB_TB
  return check_launch("rb_sparse_sign_table");
}

int sketch_sparse_sign_tab(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const int32_t* offs,
                           const uint16_t* lists, int k, int nnz, double* out, int64_t ldo, int acc, void* ws,
                           size_t wsb, cudaStream_t st) {
  const int s = std::min(nnz, k);
  RB_REQUIRE(n >= 0 && ncols >= 1 && k >= 1 && s >= 1 && s <= 16 && out && ldo >= k &&
                 (n == 0 || (X && ldx >= n && offs && lists)),
             "rb_sketch_sparse_sign_tab: bad args");
  return xd == RB_F32 ? sparse_sketch_tab<float>(n, ncols, (const float*)X, ldx, offs, lists, k, s, out, ldo, acc, ws,
                                                 wsb, st)
                      : sparse_sketch_tab<double>(n, ncols, (const double*)X, ldx, offs, lists, k, s, out, ldo, acc,
                                                  ws, wsb, st);
}

size_t gauss_tc_ws_bytes(int64_t n, int ncols, int k);
int sketch_gaussian_tc(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                       int64_t n, const uint8_t* qt, int64_t ldt, int k, double scale, double* out1, int64_t ldo1,
                       double* out2, int64_t ldo2, int acc, void* ws, size_t wsb, cudaStream_t st, bool lean = false,
                       int dig = 6, const void* pre2 = nullptr, int qpl = 2);

// [out1 | out2] = scale * (q @ [X1 | X2]).  mode 0 = auto (tensor pipe when
// every input is binary32), 1 = fp64 CUDA cores, 2 = tensor pipe, 3 = tensor
// pipe with the lean CTA (<= 64 columns; made to run beside the projection),
// 4 / 5 = tensor pipe with four / three byte digits of X per entry instead
// of six (fixed-point rounding at 2^(E-31) / 2^(E-23) of each chunk's max
// instead of 2^(E-47); 2/3 and 1/2 of the tensor work).
int sketch_gaussian2(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                     int64_t n, const uint8_t* theta, int64_t ldt, int k, double scale, double* out1, int64_t ldo1,
                     double* out2, int64_t ldo2, int acc, int mode, void* ws, size_t wsb, cudaStream_t st,
                     const void* pre2) {
  RB_REQUIRE(c1 >= 1 && c2 >= 0 && c1 <= 64 && c2 <= 64 && k >= 1 && ldo1 >= k && out1 &&
                 (c2 == 0 || (out2 && ldo2 >= k)),
             "rb_sketch_gaussian: bad args");
  RB_REQUIRE(n == 0 || (X1 && ld1 >= n && (c2 == 0 || (X2 && ld2 >= n)) && theta && ldt >= n),
             "rb_sketch_gaussian: bad X/theta");
  // mode + 16: the table's lo plane is zero (8-bit operator, rb_gaussian_fill_bits
  // with bits = 8): the tensor sketch skips it (half the table stream, half the MMAs)
  const int qpl = (mode & 16) ? 1 : 2;
  mode &= 15;
  RB_REQUIRE(mode >= 0 && mode <= 5, "rb_sketch_gaussian: bad mode %d", mode);
  const int dig = mode == 4 ? 4 : mode == 5 ? 3 : 6;
  if (mode == 3 && c1 + c2 <= 64)
    return sketch_gaussian_tc(xd1, X1, ld1, c1, xd2, X2, ld2, c2, n, theta, ldt, k, scale, out1, ldo1, out2, ldo2,
                              acc, ws, wsb, st, true);
  const bool tc = mode >= 2 || (mode == 0 && xd1 == RB_F32 && (c2 == 0 || xd2 == RB_F32));
  // > 64 columns: CTA pairs sharing the table stream (RB_TC_PAIR=0: two passes)
  static const int pair = getenv("RB_TC_PAIR") ? atoi(getenv("RB_TC_PAIR")) : 1;
  RB_REQUIRE(!pre2 || (tc && pair && c2 > 0 && c1 + c2 > 64 && mode != 3),
             "rb_sketch_gaussian2_pre: the pre-encoded input needs the paired tensor form");
  if (tc && (c1 + c2 <= 64 || (pair && c2 > 0)))
    return sketch_gaussian_tc(xd1, X1, ld1, c1, xd2, X2, ld2, c2, n, theta, ldt, k, scale, out1, ldo1, out2, ldo2,
                              acc, ws, wsb, st, false, dig, pre2, qpl);
  if (tc) {
    int rc = sketch_gaussian_tc(xd1, X1, ld1, c1, RB_F32, nullptr, 0, 0, n, theta, ldt, k, scale, out1, ldo1,
                                nullptr, 0, acc, ws, wsb, st, false, dig, nullptr, qpl);
    if (rc == RB_OK)
      rc = sketch_gaussian_tc(xd2, X2, ld2, c2, RB_F32, nullptr, 0, 0, n, theta, ldt, k, scale, out2, ldo2, nullptr,
                              0, acc, ws, wsb, st, false, dig, nullptr, qpl);
    return rc;
  }
  PlaneSrc src{theta, ldt, k};
  int rc = xd1 == RB_F32
               ? dense_sketch<float>(n, c1, (const float*)X1, ld1, src, k, scale, out1, ldo1, acc, ws, wsb, st)
               : dense_sketch<double>(n, c1, (const double*)X1, ld1, src, k, scale, out1, ldo1, acc, ws, wsb, st);
  if (rc == RB_OK && c2 > 0)
    rc = xd2 == RB_F32
             ? dense_sketch<float>(n, c2, (const float*)X2, ld2, src, k, scale, out2, ldo2, acc, ws, wsb, st)
             : dense_sketch<double>(n, c2, (const double*)X2, ld2, src, k, scale, out2, ldo2, acc, ws, wsb, st);
  return rc;
}

int sketch_gaussian(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const uint8_t* theta, int64_t ldt,
                    int k, double scale, double* out, int64_t ldo, int acc, int mode, void* ws, size_t wsb,
                    cudaStream_t st) {
  return sketch_gaussian2(xd, X, ldx, ncols, RB_F32, nullptr, 0, 0, n, theta, ldt, k, scale, out, ldo, nullptr, 0,
                          acc, mode, ws, wsb, st, nullptr);
}

int sketch_signs(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const uint32_t* bits, int64_t ldb,
                 int k, double scale, double* out, int64_t ldo, int acc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(ncols >= 1 && ncols <= 64 && k >= 1 && ldo >= k && out, "rb_sketch_signs: bad args");
  RB_REQUIRE(n == 0 || (X && ldx >= n && bits && ldb * 32 >= n), "rb_sketch_signs: bad X/bits");
  BitSrc src{bits, ldb};
  if (xd == RB_F32) return dense_sketch<float>(n, ncols, (const float*)X, ldx, src, k, scale, out, ldo, acc, ws, wsb, st);
  return dense_sketch<double>(n, ncols, (const double*)X, ldx, src, k, scale, out, ldo, acc, ws, wsb, st);
}

int sketch_srht(int xd, int64_t n, int ncols, const void* X, int64_t ldx, int64_t row0, int64_t n_pad,
                const uint32_t* bits, const int64_t* sample, int k, double scale, double* out, int64_t ldo,
                int acc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(ncols >= 1 && k >= 1 && ldo >= k && out && bits && sample, "rb_sketch_srht: bad args");
  RB_REQUIRE(n == 0 || (X && ldx >= n), "rb_sketch_srht: bad X");
  if (xd == RB_F32) return srht_sketch<float>(n, ncols, (const float*)X, ldx, row0, n_pad, bits, sample, k, scale, out, ldo, acc, ws, wsb, st);
  return srht_sketch<double>(n, ncols, (const double*)X, ldx, row0, n_pad, bits, sample, k, scale, out, ldo, acc, ws, wsb, st);
}

int sketch_sparse_sign(int xd, int64_t n, int ncols, const void* X, int64_t ldx, int64_t row0, uint64_t seed,
                       int k, int nnz, double* out, int64_t ldo, int acc, void* ws, size_t wsb, cudaStream_t st) {
  RB_REQUIRE(ncols >= 1 && k >= 1 && ldo >= k && out, "rb_sketch_sparse_sign: bad args");
  RB_REQUIRE(n == 0 || (X && ldx >= n), "rb_sketch_sparse_sign: bad X");
  if (xd == RB_F32) return sparse_sketch<float>(n, ncols, (const float*)X, ldx, row0, seed, k, nnz, out, ldo, acc, ws, wsb, st);
  return sparse_sketch<double>(n, ncols, (const double*)X, ldx, row0, seed, k, nnz, out, ldo, acc, ws, wsb, st);
}

}  // namespace rb
