// K1/K2 on the tensor pipe: the gaussian sketch  out = q @ X  (q the int16
// table of the gaussian kind) computed EXACTLY with tcgen05 kind::i8 MMAs.
//
// Exact integer split (Ozaki-style):
//   q  = 256 qh + ql,            qh = q >> 8 (s8), ql = q & 255 (u8)
//   x ~= xi 2^(E - 30)           per (column, 8192-row chunk); E: every |x| of
//                                the chunk is < 2^E; xi a signed 31-bit integer
//   xi = b3 2^24 + b2 2^16 + b1 2^8 + b0,   b3 s8, b2 b1 b0 u8
// so q xi is a sum of 8 byte products grouped by weight 2^(8g), g = 0..4.
// Each group accumulates exactly in an int32 TMEM accumulator over one chunk
// (< 2^17 per row, < 2^30 per chunk), is drained to fp64 (the groups combine
// exactly into an integer < 2^53 up to the top bits) and scaled by
// 2^(E - 30).  Relative to the fp64 reference Theta @ X the only errors are
// fp64 accumulation and the fixed-point rounding of entries far below their
// chunk's max (absolute 2^(E - 31)).
//
// Kernel (one CTA = 128 sketch rows x a run of whole chunks), warp-specialised:
//   warp 0 lane 0  producer: per 128-row K tile, ONE 32 KB bulk async copy of
//                  the q tile (both planes, pre-tiled in HBM: gauss_layout.cuh)
//                  and ONE 4 x 128 x NP byte copy of the X planes, completing
//                  on a transaction mbarrier; 3-stage ring.
//   warp 1 lane 0  MMA issuer: 16 tcgen05.mma (M=128, N=NP, K=32) per tile,
//                  tcgen05.commit frees the stage; at chunk ends commits the
//                  TMEM buffer to the epilogue (TMEM double-buffered if it fits).
//   warps 4..7     epilogue: tcgen05.ld of the 5 int32 groups of their 32
//                  lanes, exact recombination, fp64 accumulation in registers.
// The kernel is HBM-bound on the q stream (2 bytes per entry).
#include "common.cuh"
#include "gauss_layout.cuh"
#include "tc.cuh"

namespace rb {

int sm_count();

namespace {

using gl::kBK;
using gl::kTM;
constexpr int kChunk = 8192;  // rows per exact int32 accumulation
constexpr int kTPC = kChunk / kBK;
constexpr int kStages = 3;
constexpr int kThreads = 256;

// ---- pre-pass: X -> tiled byte planes + exponents ---------------------------------
// grid (nchunks, ncols), 256 threads x 32 rows (two 16-row segments each).
template <typename TX>
__global__ void __launch_bounds__(256)
split_planes(int64_t n, int ncols, int NP, const TX* __restrict__ X, int64_t ldx, uint8_t* __restrict__ planes,
             int* __restrict__ exps) {
  __shared__ float red[8];
  const int c = blockIdx.x, j = blockIdx.y;
  const int64_t base = (int64_t)c * kChunk;
  const TX* xc = X + (int64_t)j * ldx;
  // thread t owns rows base + 16 (t + 256 u) + e, u = 0..1, e = 0..15
  double v[2][16];
  float mx = 0.f;
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int64_t i = base + 16 * (threadIdx.x + 256 * u) + e;
      v[u][e] = i < n ? (double)xc[i] : 0.0;
      mx = fmaxf(mx, (float)fabs(v[u][e]));
    }
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  float m = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) m = fmaxf(m, red[w]);
  int E = 0;
  if (m > 0.f) frexpf(m, &E);  // m < 2^E; float rounding is monotone, so every |x| < 2^E
  if (threadIdx.x == 0) exps[(int64_t)c * NP + j] = E;
  const double s = ldexp(1.0, 30 - E);
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    const int64_t i0 = base + 16 * (threadIdx.x + 256 * u);
    uint32_t w[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t xi = (uint32_t)(int)rint(v[u][4 * q + e] * s);
        b0 |= (xi & 255u) << (8 * e);
        b1 |= ((xi >> 8) & 255u) << (8 * e);
        b2 |= ((xi >> 16) & 255u) << (8 * e);
        b3 |= ((xi >> 24) & 255u) << (8 * e);
      }
      w[0][q] = b0;
      w[1][q] = b1;
      w[2][q] = b2;
      w[3][q] = b3;
    }
#pragma unroll
    for (int pl = 0; pl < 4; ++pl)
      *reinterpret_cast<uint4*>(planes + gl::x_offset(pl, j, i0, NP)) = make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]);
  }
}

// zero the padding columns j in [ncols, NP) of every tile
__global__ void zero_pad_cols(int64_t ktiles, int ncols, int NP, uint8_t* __restrict__ planes) {
  const int64_t kt = blockIdx.x;
  if (kt >= ktiles) return;
  for (int e = threadIdx.x; e < 4 * (kBK / 16) * (NP - ncols); e += blockDim.x) {
    const int pl = e / ((kBK / 16) * (NP - ncols));
    const int rem = e % ((kBK / 16) * (NP - ncols));
    const int kc = rem / (NP - ncols), j = ncols + rem % (NP - ncols);
    *reinterpret_cast<uint4*>(planes + gl::x_offset(pl, j, kt * kBK + kc * 16, NP)) = make_uint4(0, 0, 0, 0);
  }
}

template <int NP>
struct Smem {
  uint8_t a[kStages][2][kBK / 16][kTM][16];  // one q tile
  uint8_t b[kStages][4][kBK / 16][NP][16];   // one X-plane tile
  uint64_t full[kStages], empty[kStages];
  uint64_t tfull[2], tempty[2];
  uint32_t tbase;
};

template <int NP>
__global__ void __launch_bounds__(kThreads, 1)
gauss_tc_partial(int64_t n, int ncols, const uint8_t* __restrict__ qt, int64_t ldt, int k,
                 const uint8_t* __restrict__ planes, const int* __restrict__ exps, int nchunks, int chunks_per_cta,
                 double* __restrict__ ws) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NP>& S = *reinterpret_cast<Smem<NP>*>(smem_raw);
  constexpr int kGroupCols = 5 * NP;
  constexpr int kBufs = (2 * kGroupCols <= 512) ? 2 : 1;
  constexpr uint32_t kAlloc = kBufs * kGroupCols <= 64 ? 64 : kBufs * kGroupCols <= 128 ? 128
                              : kBufs * kGroupCols <= 256 ? 256 : 512;
  constexpr uint32_t kABytes = 2 * kTM * kBK, kBBytes = 4 * kBK * NP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x;
  const int c_beg = blockIdx.y * chunks_per_cta;
  const int c_end = min(nchunks, c_beg + chunks_per_cta);
  const int64_t KT = ldt / kBK;
  const int64_t kt_beg = (int64_t)c_beg * kTPC;
  const int64_t kt_end = min((int64_t)c_end * kTPC, (n + kBK - 1) / kBK);
  const int T = (int)(kt_end - kt_beg);

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&S.full[s], 1);
      tc::mbar_init(&S.empty[s], 1);
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

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint8_t* qtile = qt + (int64_t)mt * KT * 2 * gl::kTileBytes;
      for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        if (t >= kStages) tc::mbar_wait(&S.empty[s], ((t / kStages) - 1) & 1);
        const int64_t kt = kt_beg + t;
        tc::mbar_arrive_expect_tx(&S.full[s], kABytes + kBBytes);
        tc::bulk_g2s(&S.a[s][0][0][0][0], qtile + kt * 2 * gl::kTileBytes, kABytes, &S.full[s]);
        tc::bulk_g2s(&S.b[s][0][0][0][0], planes + kt * (int64_t)kBBytes, kBBytes, &S.full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t ID_SS = tc::idesc_i8(kTM, NP, true, true);
      constexpr uint32_t ID_SU = tc::idesc_i8(kTM, NP, true, false);
      constexpr uint32_t ID_US = tc::idesc_i8(kTM, NP, false, true);
      constexpr uint32_t ID_UU = tc::idesc_i8(kTM, NP, false, false);
      int chunk_i = 0;
      for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        const int tin = t % kTPC;
        const int buf = chunk_i % kBufs;
        if (tin == 0 && chunk_i >= kBufs) tc::mbar_wait(&S.tempty[buf], ((chunk_i / kBufs) - 1) & 1);
        tc::mbar_wait(&S.full[s], (t / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t d = tbase + buf * kGroupCols;
#pragma unroll
        for (int ks = 0; ks < kBK / 32; ++ks) {
          const uint32_t acc = (tin == 0 && ks == 0) ? 0u : 1u;
          const uint64_t ah = tc::sdesc_kmajor(tc::smem_u32(&S.a[s][0][2 * ks][0][0]), kTM * 16, 128);
          const uint64_t al = tc::sdesc_kmajor(tc::smem_u32(&S.a[s][1][2 * ks][0][0]), kTM * 16, 128);
          uint64_t b[4];
#pragma unroll
          for (int pl = 0; pl < 4; ++pl)
            b[pl] = tc::sdesc_kmajor(tc::smem_u32(&S.b[s][pl][2 * ks][0][0]), NP * 16, 128);
          tc::mma_i8(d + 4 * NP, ah, b[3], ID_SS, acc);  // 2^32
          tc::mma_i8(d + 3 * NP, ah, b[2], ID_SU, acc);  // 2^24
          tc::mma_i8(d + 3 * NP, al, b[3], ID_US, 1u);
          tc::mma_i8(d + 2 * NP, ah, b[1], ID_SU, acc);  // 2^16
          tc::mma_i8(d + 2 * NP, al, b[2], ID_UU, 1u);
          tc::mma_i8(d + 1 * NP, ah, b[0], ID_SU, acc);  // 2^8
          tc::mma_i8(d + 1 * NP, al, b[1], ID_UU, 1u);
          tc::mma_i8(d + 0 * NP, al, b[0], ID_UU, acc);  // 2^0
        }
        tc::mma_commit(&S.empty[s]);
        if (tin == kTPC - 1 || t == T - 1) {
          tc::mma_commit(&S.tfull[buf]);
          ++chunk_i;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp - 4;  // TMEM lane quadrant
    const int row = q * 32 + lane;
    double acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = 0.0;
    const int nch = c_end - c_beg;
    const int nch_here = (T + kTPC - 1) / kTPC;
    for (int ci = 0; ci < nch_here && ci < nch; ++ci) {
      const int buf = ci % kBufs;
      tc::mbar_wait(&S.tfull[buf], (ci / kBufs) & 1);
      tc::tc_fence_after();
      const uint32_t la = tbase + ((uint32_t)(q * 32) << 16) + buf * kGroupCols;
      const int* ex = exps + (int64_t)(c_beg + ci) * NP;
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 16) {
        uint32_t g[5][16];
#pragma unroll
        for (int gi = 0; gi < 5; ++gi) tc::tmem_ld16(la + gi * NP + c0, g[gi]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          double v = (double)(int)g[4][jj];
          v = v * 256.0 + (double)(int)g[3][jj];
          v = v * 256.0 + (double)(int)g[2][jj];
          v = v * 256.0 + (double)(int)g[1][jj];
          v = v * 256.0 + (double)(int)g[0][jj];
          acc[c0 + jj] += ldexp(v, ex[c0 + jj] - 30);
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[buf]);
    }
    // partial: ws[split][j][r]
    const int r = mt * kTM + row;
    double* dst = ws + (int64_t)blockIdx.y * k * ncols;
    if (r < k) {
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (j < ncols) dst[r + (int64_t)j * k] = acc[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tbase, kAlloc);
}

__global__ void reduce_splits_tc(const double* __restrict__ ws, int splits, int k, int ncols, double scale,
                                 double* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)k * ncols;
  if (e >= tot) return;
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += ws[(int64_t)q * tot + e];
  const int r = (int)(e % k), j = (int)(e / k);
  double* o = out + r + (int64_t)j * ldo;
  *o = accumulate ? *o + scale * s : scale * s;
}

int np_for(int ncols) { return ncols <= 16 ? 16 : ncols <= 32 ? 32 : ncols <= 48 ? 48 : 64; }

template <int NP>
int launch_np(int64_t n, int ncols, const uint8_t* qt, int64_t ldt, int k, const uint8_t* planes, const int* exps,
              int nchunks, double* part, size_t part_bytes, int* splits_out, cudaStream_t st) {
  const int mt = ceil_div(k, kTM);
  int splits = std::max(1, std::min(nchunks, (sm_count() + mt - 1) / mt));
  const size_t per = (size_t)k * ncols * sizeof(double);
  if ((size_t)splits * per > part_bytes) splits = (int)std::max<size_t>(1, part_bytes / per);
  RB_REQUIRE((size_t)splits * per <= part_bytes, "gaussian tc: workspace too small");
  const int cpc = ceil_div(nchunks, splits);
  splits = ceil_div(nchunks, cpc);
  const size_t smem = sizeof(Smem<NP>) + 1024;
  cudaFuncSetAttribute(gauss_tc_partial<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  RB_KLAUNCH gauss_tc_partial<NP><<<dim3(mt, splits), kThreads, smem, st>>>(n, ncols, qt, ldt, k, planes, exps,
                                                                           nchunks, cpc, part);
  *splits_out = splits;
  return check_launch("gauss_tc_partial");
}

}  // namespace

size_t gauss_tc_ws_bytes(int64_t n, int ncols, int k) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const size_t planes = (size_t)4 * 64 * nchunks * kChunk;
  const size_t exps = ((size_t)64 * nchunks * sizeof(int) + 255) / 256 * 256;
  const size_t part = (size_t)(sm_count() + 1) * std::max(k, 64) * std::max(ncols, 1) * sizeof(double);
  return planes + exps + part + 1024;
}

// out = scale * (q @ X) on the tensor pipe; X binary32 or binary64 (n x ncols).
int sketch_gaussian_tc(int xd, int64_t n, int ncols, const void* X, int64_t ldx, const uint8_t* qt, int64_t ldt,
                       int k, double scale, double* out, int64_t ldo, int acc, void* ws, size_t wsb,
                       cudaStream_t st) {
  RB_REQUIRE(ncols >= 1 && ncols <= 64 && k >= 1 && ldo >= k && out, "rb_sketch_gaussian (tensor): bad args");
  RB_REQUIRE(n == 0 || (X && ldx >= n && qt && ldt >= n && ldt % kBK == 0),
             "rb_sketch_gaussian (tensor): bad X/theta (ldt %% 128 required)");
  const int NP = np_for(ncols);
  const int nchunks = (int)((n + kChunk - 1) / kChunk);
  const int64_t ktiles = (int64_t)nchunks * kTPC;
  const size_t planes_b = (size_t)ktiles * 4 * kBK * NP;
  const size_t exps_b = ((size_t)NP * nchunks * sizeof(int) + 255) / 256 * 256;
  RB_REQUIRE(ws && wsb > planes_b + exps_b + 1024, "rb_sketch_gaussian (tensor): workspace too small");
  uint8_t* planes = (uint8_t*)ws;
  int* exps = (int*)((uint8_t*)ws + planes_b);
  double* part = (double*)((uint8_t*)ws + planes_b + exps_b);
  const size_t part_b = wsb - planes_b - exps_b;
  int splits = 0;
  if (n > 0) {
    dim3 g(nchunks, ncols);
    if (xd == RB_F32)
      RB_KLAUNCH split_planes<float><<<g, 256, 0, st>>>(n, ncols, NP, (const float*)X, ldx, planes, exps);
    else
      RB_KLAUNCH split_planes<double><<<g, 256, 0, st>>>(n, ncols, NP, (const double*)X, ldx, planes, exps);
    if (NP > ncols) RB_KLAUNCH zero_pad_cols<<<(unsigned)ktiles, 256, 0, st>>>(ktiles, ncols, NP, planes);
    int rc;
    if (NP == 16) rc = launch_np<16>(n, ncols, qt, ldt, k, planes, exps, nchunks, part, part_b, &splits, st);
    else if (NP == 32) rc = launch_np<32>(n, ncols, qt, ldt, k, planes, exps, nchunks, part, part_b, &splits, st);
    else if (NP == 48) rc = launch_np<48>(n, ncols, qt, ldt, k, planes, exps, nchunks, part, part_b, &splits, st);
    else rc = launch_np<64>(n, ncols, qt, ldt, k, planes, exps, nchunks, part, part_b, &splits, st);
    if (rc != RB_OK) return rc;
  }
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits_tc<<<ceil_div(tot, 256), 256, 0, st>>>(part, splits, k, ncols, scale, out, ldo, acc);
  return check_launch("rb_sketch_gaussian (tensor)");
}

}  // namespace rb
