// K1/K2 on the tensor pipe: the gaussian sketch  out = q @ [X1 | X2]  (q the
// int16 table of the gaussian kind) computed EXACTLY with tcgen05 kind::i8.
//
// Exact integer split (Ozaki-style):
//   q  = 256 qh + ql,            qh = q >> 8 (s8), ql = q & 255 (u8)
//   x ~= xi 2^(E - 30)           per (column, 8192-row chunk); E: every |x| of
//                                the chunk is < 2^E; xi a signed 31-bit integer
//   xi = b3 2^24 + b2 2^16 + b1 2^8 + b0,   b3 s8, b2 b1 b0 u8
// so q xi is a sum of 8 byte products grouped by weight 2^(8g), g = 0..4.
// Each group accumulates exactly in an int32 TMEM accumulator over one chunk
// (< 2^17 per row, < 2^30 per chunk), is drained to fp64 and scaled by
// 2^(E - 30).  Relative to the fp64 reference Theta @ X the only errors are
// fp64 accumulation and the fixed-point rounding of entries far below their
// chunk's max (absolute 2^(E - 31)).
//
// Two inputs: the sweep sketches [Q'_i | W_(i+1)] in ONE pass so the q stream
// (2 bytes per entry, the dominant HBM traffic) is read once per block.
//
// Kernel (one CTA = 128 sketch rows x a contiguous run of 128-row K tiles),
// warp-specialised:
//   warp 0 lane 0  producer: per K tile ONE bulk async copy of the q tile
//                  (32 KB, pre-tiled in HBM: gauss_layout.cuh) and ONE of the
//                  X-plane tile (4 x 128 x NP bytes) onto a transaction
//                  mbarrier; 3-stage ring (2 for NP > 64).
//   warp 1 lane 0  MMA issuer: 16 tcgen05.mma (M=128, N=NP, K=32) per tile;
//                  tcgen05.commit frees the stage; at chunk ends hands the
//                  TMEM buffer to the epilogue (double-buffered if it fits).
//   warps 4..7     epilogue: tcgen05.ld of the 5 int32 groups of their 32
//                  lanes, exact recombination, fp64 scale-and-add into the
//                  CTA's own slice of the split-K partial buffer (L2-resident).
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
constexpr int kThreads = 256;

template <int NP>
constexpr int stages_for() { return NP <= 64 ? 3 : 2; }

// ---- pre-pass: [X1 | X2] -> tiled byte planes + exponents --------------------------
// grid (nchunks, NP / 2): one CTA per chunk x column pair; thread t owns 32
// consecutive rows of both columns, so every plane store is a full 32-byte
// sector (the two columns' 16-byte segments are adjacent in the layout).
// Columns >= ncols are written as zeros (the UMMA N padding).
template <typename T1, typename T2>
__global__ void __launch_bounds__(256)
split_planes(int64_t n, int c1, const T1* __restrict__ X1, int64_t ld1, int c2, const T2* __restrict__ X2,
             int64_t ld2, int NP, uint8_t* __restrict__ planes, int* __restrict__ exps) {
  __shared__ float red[2][8];
  const int c = blockIdx.x;
  const int j0 = 2 * blockIdx.y;
  const int64_t base = (int64_t)c * kChunk + 32 * threadIdx.x;
  double v[2][32];
  float mx[2] = {0.f, 0.f};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = j0 + h;
    if (j < c1) {
      const T1* x = X1 + (int64_t)j * ld1;
#pragma unroll
      for (int e = 0; e < 32; ++e) v[h][e] = base + e < n ? (double)x[base + e] : 0.0;
    } else if (j < c1 + c2) {
      const T2* x = X2 + (int64_t)(j - c1) * ld2;
#pragma unroll
      for (int e = 0; e < 32; ++e) v[h][e] = base + e < n ? (double)x[base + e] : 0.0;
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) v[h][e] = 0.0;
    }
#pragma unroll
    for (int e = 0; e < 32; ++e) mx[h] = fmaxf(mx[h], (float)fabs(v[h][e]));
    for (int o = 16; o; o >>= 1) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], o));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mx[0];
    red[1][threadIdx.x >> 5] = mx[1];
  }
  __syncthreads();
  double s[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float m = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = fmaxf(m, red[h][w]);
    int E = 0;
    if (m > 0.f) frexpf(m, &E);  // m < 2^E; float rounding is monotone, so every |x| < 2^E
    if (threadIdx.x == 0) exps[(int64_t)c * NP + j0 + h] = E;
    s[h] = ldexp(1.0, 30 - E);
  }
#pragma unroll
  for (int seg = 0; seg < 2; ++seg) {
    uint32_t w[4][2][4];  // [plane][column][word]
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t xi = (uint32_t)(int)rint(v[h][16 * seg + 4 * q + e] * s[h]);
          b0 |= (xi & 255u) << (8 * e);
          b1 |= ((xi >> 8) & 255u) << (8 * e);
          b2 |= ((xi >> 16) & 255u) << (8 * e);
          b3 |= ((xi >> 24) & 255u) << (8 * e);
        }
        w[0][h][q] = b0;
        w[1][h][q] = b1;
        w[2][h][q] = b2;
        w[3][h][q] = b3;
      }
    const int64_t i0 = base + 16 * seg;
#pragma unroll
    for (int pl = 0; pl < 4; ++pl) {
      uint4* dst = reinterpret_cast<uint4*>(planes + gl::x_offset(pl, j0, i0, NP));
      dst[0] = make_uint4(w[pl][0][0], w[pl][0][1], w[pl][0][2], w[pl][0][3]);
      dst[1] = make_uint4(w[pl][1][0], w[pl][1][1], w[pl][1][2], w[pl][1][3]);
    }
  }
}

template <int NP>
struct Smem {
  static constexpr int S = stages_for<NP>();
  uint8_t a[S][2][kBK / 16][kTM][16];  // one q tile
  uint8_t b[S][4][kBK / 16][NP][16];   // one X-plane tile
  uint64_t full[S], empty[S];
  uint64_t tfull[2], tempty[2];
  uint32_t tbase;
};

template <int NP>
__global__ void __launch_bounds__(kThreads, 1)
gauss_tc_partial(int64_t n, int ncols, const uint8_t* __restrict__ qt, int64_t ldt, int k,
                 const uint8_t* __restrict__ planes, const int* __restrict__ exps, int tiles_per_cta,
                 double* __restrict__ ws) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NP>& S = *reinterpret_cast<Smem<NP>*>(smem_raw);
  constexpr int kStages = Smem<NP>::S;
  constexpr int kGroupCols = 5 * NP;
  constexpr int kBufs = (2 * kGroupCols <= 512) ? 2 : 1;
  constexpr uint32_t kAlloc = kBufs * kGroupCols <= 64 ? 64 : kBufs * kGroupCols <= 128 ? 128
                              : kBufs * kGroupCols <= 256 ? 256 : 512;
  static_assert(kGroupCols <= 512, "TMEM: 5 groups x NP columns must fit 512");
  constexpr uint32_t kABytes = 2 * kTM * kBK, kBBytes = 4 * kBK * NP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x;
  const int64_t KT = ldt / kBK;
  // this CTA's K tiles [kt_beg, kt_end); accumulators drain at every global
  // 8192-row chunk boundary and at kt_end (segments)
  const int64_t kt_beg = (int64_t)blockIdx.y * tiles_per_cta;
  const int64_t kt_end = min(kt_beg + tiles_per_cta, (n + kBK - 1) / kBK);
  const int T = kt_end > kt_beg ? (int)(kt_end - kt_beg) : 0;

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
      int seg_i = 0;
      for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        const int64_t kt = kt_beg + t;
        const bool seg_first = (t == 0) || (kt % kTPC == 0);
        const bool seg_last = (t == T - 1) || ((kt + 1) % kTPC == 0);
        const int buf = seg_i % kBufs;
        if (seg_first && seg_i >= kBufs) tc::mbar_wait(&S.tempty[buf], ((seg_i / kBufs) - 1) & 1);
        tc::mbar_wait(&S.full[s], (t / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t d = tbase + buf * kGroupCols;
#pragma unroll
        for (int ks = 0; ks < kBK / 32; ++ks) {
          const uint32_t acc = (seg_first && ks == 0) ? 0u : 1u;
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
        if (seg_last) {
          tc::mma_commit(&S.tfull[buf]);
          ++seg_i;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int q = warp - 4;  // TMEM lane quadrant
    const int r = mt * kTM + q * 32 + lane;
    double* dst = ws + (int64_t)blockIdx.y * k * ncols + r;
    int ci = 0;
    for (int64_t ks = kt_beg; ks < kt_end; ++ci) {
      const int64_t chunk = ks / kTPC;
      ks = min(kt_end, (chunk + 1) * kTPC);
      const int buf = ci % kBufs;
      tc::mbar_wait(&S.tfull[buf], (ci / kBufs) & 1);
      tc::tc_fence_after();
      const uint32_t la = tbase + ((uint32_t)(q * 32) << 16) + buf * kGroupCols;
      const int* ex = exps + chunk * NP;
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 16) {
        uint32_t g[5][16];
#pragma unroll
        for (int gi = 0; gi < 5; ++gi) tc::tmem_ld16(la + gi * NP + c0, g[gi]);
        tc::tmem_ld_wait();
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = c0 + jj;
          if (j < ncols && r < k) {
            double v = (double)(int)g[4][jj];
            v = v * 256.0 + (double)(int)g[3][jj];
            v = v * 256.0 + (double)(int)g[2][jj];
            v = v * 256.0 + (double)(int)g[1][jj];
            v = v * 256.0 + (double)(int)g[0][jj];
            v = ldexp(v, ex[j] - 30);
            double* o = dst + (int64_t)j * k;
            *o = ci ? *o + v : v;
          }
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[buf]);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tbase, kAlloc);
}

__global__ void reduce_splits_tc(const double* __restrict__ ws, int splits, int k, int c1, int ncols, double scale,
                                 double* __restrict__ out1, int64_t ldo1, double* __restrict__ out2, int64_t ldo2,
                                 int accumulate) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)k * ncols;
  if (e >= tot) return;
  double s = 0.0;
  for (int q = 0; q < splits; ++q) s += ws[(int64_t)q * tot + e];
  const int r = (int)(e % k), j = (int)(e / k);
  double* o = j < c1 ? out1 + r + (int64_t)j * ldo1 : out2 + r + (int64_t)(j - c1) * ldo2;
  *o = accumulate ? *o + scale * s : scale * s;
}

int np_for(int ncols) { return ncols <= 16 ? 16 : ncols <= 32 ? 32 : ncols <= 48 ? 48 : ncols <= 64 ? 64 : ncols <= 80 ? 80 : 96; }

template <int NP>
int launch_np(int64_t n, int ncols, const uint8_t* qt, int64_t ldt, int k, const uint8_t* planes, const int* exps,
              double* part, size_t part_bytes, int* splits_out, cudaStream_t st) {
  const int mt = ceil_div(k, kTM);
  // one wave: floor(SMs / m-tiles) K ranges of equal tile counts
  const int64_t ktn = (n + kBK - 1) / kBK;
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(ktn, sm_count() / mt));
  const size_t per = (size_t)k * ncols * sizeof(double);
  if ((size_t)splits * per > part_bytes) splits = (int)std::max<size_t>(1, part_bytes / per);
  RB_REQUIRE((size_t)splits * per <= part_bytes, "gaussian tc: workspace too small");
  const int tpc = (int)((ktn + splits - 1) / splits);
  splits = (int)((ktn + tpc - 1) / tpc);
  const size_t smem = sizeof(Smem<NP>) + 1024;
  cudaFuncSetAttribute(gauss_tc_partial<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  RB_KLAUNCH gauss_tc_partial<NP><<<dim3(mt, splits), kThreads, smem, st>>>(n, ncols, qt, ldt, k, planes, exps, tpc,
                                                                           part);
  *splits_out = splits;
  return check_launch("gauss_tc_partial");
}

template <typename T1>
void launch_split(int xd2, dim3 g, int64_t n, int c1, const void* X1, int64_t ld1, int c2, const void* X2, int64_t ld2,
                  int NP, uint8_t* planes, int* exps, cudaStream_t st) {
  if (xd2 == RB_F32)
    RB_KLAUNCH split_planes<T1, float><<<g, 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const float*)X2, ld2, NP,
                                                         planes, exps);
  else
    RB_KLAUNCH split_planes<T1, double><<<g, 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const double*)X2, ld2, NP,
                                                          planes, exps);
}

}  // namespace

size_t gauss_tc_ws_bytes(int64_t n, int ncols, int k) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const int cols = std::max(ncols, 1) <= 48 ? 96 : 96;  // room for a fused two-input call
  const size_t planes = (size_t)4 * cols * nchunks * kChunk;
  const size_t exps = ((size_t)cols * nchunks * sizeof(int) + 255) / 256 * 256;
  const size_t part = (size_t)(sm_count() + 1) * std::max(k, 64) * cols * sizeof(double);
  return planes + exps + part + 1024;
}

// [out1 | out2] = scale * (q @ [X1 | X2]) on the tensor pipe; each X is
// binary32 or binary64 (n rows); c2 may be 0.
int sketch_gaussian_tc(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                       int64_t n, const uint8_t* qt, int64_t ldt, int k, double scale, double* out1, int64_t ldo1,
                       double* out2, int64_t ldo2, int acc, void* ws, size_t wsb, cudaStream_t st) {
  const int ncols = c1 + c2;
  RB_REQUIRE(c1 >= 1 && c2 >= 0 && ncols <= 96 && k >= 1 && ldo1 >= k && out1 && (c2 == 0 || (out2 && ldo2 >= k)),
             "rb_sketch_gaussian (tensor): bad args (c1 %d, c2 %d)", c1, c2);
  RB_REQUIRE(n == 0 || (X1 && ld1 >= n && (c2 == 0 || (X2 && ld2 >= n)) && qt && ldt >= n && ldt % kBK == 0),
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
    dim3 g(nchunks, NP / 2);
    if (xd1 == RB_F32) launch_split<float>(xd2, g, n, c1, X1, ld1, c2, X2, ld2, NP, planes, exps, st);
    else launch_split<double>(xd2, g, n, c1, X1, ld1, c2, X2, ld2, NP, planes, exps, st);
    int rc;
    switch (NP) {
      case 16: rc = launch_np<16>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
      case 32: rc = launch_np<32>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
      case 48: rc = launch_np<48>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
      case 64: rc = launch_np<64>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
      case 80: rc = launch_np<80>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
      default: rc = launch_np<96>(n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st); break;
    }
    if (rc != RB_OK) return rc;
  }
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits_tc<<<ceil_div(tot, 256), 256, 0, st>>>(part, splits, k, c1, ncols, scale, out1, ldo1, out2,
                                                                  ldo2, acc);
  return check_launch("rb_sketch_gaussian (tensor)");
}

}  // namespace rb
