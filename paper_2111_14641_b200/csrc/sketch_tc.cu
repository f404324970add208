// K1/K2 on the tensor pipe: the gaussian sketch  out = q @ [X1 | X2]  (q the
// int16 table of the gaussian kind) computed EXACTLY with tcgen05 kind::i8.
//
// Exact integer split (Ozaki-style):
//   q  = 256 qh + ql,            qh = q >> 8 (s8), ql = q & 255 (u8)
//   x ~= xi 2^(E - 46)           per (column, 16384-row chunk); E: every |x|
//                                of the chunk is < 2^E; xi a signed integer,
//                                |xi| <= 2^46
//   xi = b5 2^40 + b4 2^32 + .. + b1 2^8 + b0,  balanced signed digits (s8)
// so q xi is a sum of 12 byte products grouped by weight 2^(8w), w = 0..6.
// One MMA multiplies qh by the six digit planes side by side (N = 6 NG),
// a second multiplies ql by the same operand into TMEM shifted by one block,
// so each TMEM block accumulates one weight exactly in int32 over one chunk
// (< 2^16 per row, < 2^30 per chunk).  Blocks are drained to fp64 (int64
// partial sums, two roundings) and scaled by 2^(E - 46).  Relative to the
// fp64 reference Theta @ X the only errors are fp64 accumulation and the
// fixed-point rounding of entries more than 2^22 below their chunk's max
// (absolute 2^(E - 47)): a binary32 entry within 22 binades of the max is
// exact, so the sketch carries binary64 accuracy like the CUDA-core path.
// Why six digits: Step 3 rounds X to binary32 (kernels.py:192-199), so an
// error of the sketch far below binary32 resolution still flips roundings
// of X and moves R through the cancellation of the trig family: four digits
// (2^(E-31)) drifted 4e-5 and five (2^(E-39)) 1.4e-5 / 3.1e-5 from the
// oracle on C2 samples, the binary64 path 7e-7 / 1.6e-7.
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
//   warps 4..7     epilogue: tcgen05.ld of the 7 int32 weight blocks of their
//                  32 lanes, exact recombination, fp64 scale-and-add into the
//                  CTA's own slice of the split-K partial buffer (L2-resident).
// Pre-pass (chunk_max + encode_planes): chunk exponents, then the six byte
// planes in the tiled B-operand layout (gauss_layout.cuh).
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "gauss_layout.cuh"
#include "tc.cuh"

namespace rb {

int sm_count();

namespace {

using gl::kBK;
using gl::kTM;
constexpr int kChunk = 16384;  // rows per exact int32 accumulation (< 2^16 per row, balanced digits)
constexpr int kTPC = kChunk / kBK;
constexpr int kThreads = 256;
constexpr int kSplitThreads = 256;                    // split pre-pass: one chunk x column pair per CTA
constexpr int kSplitSeg = kChunk / (16 * kSplitThreads);  // 16-row segments per thread

// pipeline depth: as many 128-row stages as fit next to each other in
// shared memory (overridable with RB_TC_STAGES for measurement)
template <int NP, int DIG = gl::kXDig>
constexpr int max_stages() { return (227 * 1024 - 2048) / (2 * kTM * kBK + DIG * kBK * NP); }

// ---- pre-pass: [X1 | X2] -> tiled byte planes + exponents --------------------------
// grid (nchunks, NP / 2): one CTA per chunk x column pair; thread t owns 32
// consecutive rows of both columns (vector loads when aligned), so every
// plane store is a full 32-byte sector (the two columns' 16-byte segments
// are adjacent in the layout).  Columns >= ncols are written as zeros (the
// UMMA N padding).  The scaling x 2^(46-E) is exact in binary64 and
// |xi| <= 2^46: binary32 entries within 22 binades of the chunk max convert
// exactly, the rest (and binary64 inputs) round once to nearest.
// L2 policy of the binary32 vector loads: the max pass keeps the chunk in L2
// (evict_last) for the encode pass, which reads it for the last time
// (evict_first) -- without the hint ncu saw 60% of the re-read miss L2.
template <int POL>
__device__ __forceinline__ float4 ld_f4(const float4* p) {
  float4 f;
  if constexpr (POL == 1 || POL == 2) {
    uint64_t pol;
    if constexpr (POL == 1)
      asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(f.x), "=f"(f.y), "=f"(f.z), "=f"(f.w) : "l"(p), "l"(pol));
  } else {
    f = __ldg(p);
  }
  return f;
}

template <int L, typename T, typename TV, int POL = 0>
__device__ __forceinline__ void loadL(const T* __restrict__ x, int64_t base, int64_t n, bool vec, TV (&v)[L]) {
  if (vec && base + L <= n) {
    if constexpr (sizeof(T) == 4) {
      const float4* p4 = reinterpret_cast<const float4*>(x + base);
#pragma unroll
      for (int q = 0; q < L / 4; ++q) {
        const float4 f = ld_f4<POL>(p4 + q);
        v[4 * q] = f.x;
        v[4 * q + 1] = f.y;
        v[4 * q + 2] = f.z;
        v[4 * q + 3] = f.w;
      }
    } else {
      const double2* p2 = reinterpret_cast<const double2*>(x + base);
#pragma unroll
      for (int q = 0; q < L / 2; ++q) {
        const double2 f = __ldg(p2 + q);
        v[2 * q] = (TV)f.x;
        v[2 * q + 1] = (TV)f.y;
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < L; ++e) v[e] = base + e < n ? (TV)x[base + e] : TV(0);
  }
}

// x 2^(46 - E) rounded to an integer (|xi| <= 2^46): the scaling is exact in
// binary64 (binary32 embeds exactly), so this is the one rounding.  For a
// binary32 x and 2^(46 - E) a normal binary32 (fast), the binary32 product is
// exact too (|x 2^(46-E)| < 2^46; a product below 2^-126 rounds to integer 0
// either way), so the binary32 path gives the same integer with no FP64 op.
struct Scale {
  double s;
  float sf;
  bool fast;
};
__device__ __forceinline__ long long fixed_of(float v, const Scale& s) {
  return s.fast ? __float2ll_rn(__fmul_rn(v, s.sf)) : __double2ll_rn((double)v * s.s);
}
__device__ __forceinline__ long long fixed_of(double v, const Scale& s) { return __double2ll_rn(v * s.s); }

// Balanced signed byte digits: xi = b5 2^40 + b4 2^32 + .. + b1 2^8 + b0
// with b0..b4 in [-128, 127] and |b5| <= 65 (|xi| <= 2^46), so every plane
// is s8 and ONE MMA can take all six planes as its B operand.  Plane order
// in the layout: 0 = b5, .., 5 = b0 (descending weight).
// Computed without a digit loop: y = xi + 0x80_8080_8080 has the unsigned
// bytes b_q + 128 (q < 5) and y >> 40 = b5 (the balanced representation is
// unique, so these are the digits), i.e. byte q of y XOR 0x80 is b_q and
// byte 5 of y is b5.  Four entries' words are byte-transposed into one word
// per plane (entry e in byte e).
__device__ __forceinline__ void planes4(const long long (&xi)[4], uint32_t (&pw)[gl::kXDig]) {
  uint32_t lo[4], hi[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const unsigned long long y = (unsigned long long)xi[e] + 0x8080808080ull;
    lo[e] = (uint32_t)y;
    hi[e] = (uint32_t)(y >> 32);
  }
  const uint32_t t01l = __byte_perm(lo[0], lo[1], 0x5140), t01h = __byte_perm(lo[0], lo[1], 0x7362);
  const uint32_t t23l = __byte_perm(lo[2], lo[3], 0x5140), t23h = __byte_perm(lo[2], lo[3], 0x7362);
  const uint32_t u01 = __byte_perm(hi[0], hi[1], 0x5140), u23 = __byte_perm(hi[2], hi[3], 0x5140);
  pw[5] = __byte_perm(t01l, t23l, 0x5410) ^ 0x80808080u;  // b0
  pw[4] = __byte_perm(t01l, t23l, 0x7632) ^ 0x80808080u;  // b1
  pw[3] = __byte_perm(t01h, t23h, 0x5410) ^ 0x80808080u;  // b2
  pw[2] = __byte_perm(t01h, t23h, 0x7632) ^ 0x80808080u;  // b3
  pw[1] = __byte_perm(u01, u23, 0x5410) ^ 0x80808080u;    // b4
  pw[0] = __byte_perm(u01, u23, 0x7632);                  // b5
}

// DIG < 6: the same construction on the (8 DIG - 2)-bit fixed point,
// y = xi + 0x80..80 (DIG - 1 bytes); plane 0 = the top digit.
template <int DIG>
__device__ __forceinline__ void planes4d(const long long (&xi)[4], uint32_t (&pw)[DIG]) {
  if constexpr (DIG == gl::kXDig) {
    planes4(xi, pw);
  } else {
    static_assert(DIG == 3 || DIG == 4, "digit counts: 6, 4, 3");
    constexpr uint32_t kBias = DIG == 4 ? 0x808080u : 0x8080u;
    uint32_t y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) y[e] = (uint32_t)(int)xi[e] + kBias;  // |xi| <= 2^(8 DIG - 2): fits 32 bits
    const uint32_t t01l = __byte_perm(y[0], y[1], 0x5140), t01h = __byte_perm(y[0], y[1], 0x7362);
    const uint32_t t23l = __byte_perm(y[2], y[3], 0x5140), t23h = __byte_perm(y[2], y[3], 0x7362);
    const uint32_t d0 = __byte_perm(t01l, t23l, 0x5410), d1 = __byte_perm(t01l, t23l, 0x7632);
    const uint32_t d2 = __byte_perm(t01h, t23h, 0x5410), d3 = __byte_perm(t01h, t23h, 0x7632);
    if constexpr (DIG == 4) {
      pw[3] = d0 ^ 0x80808080u;
      pw[2] = d1 ^ 0x80808080u;
      pw[1] = d2 ^ 0x80808080u;
      pw[0] = d3;
    } else {
      pw[2] = d0 ^ 0x80808080u;
      pw[1] = d1 ^ 0x80808080u;
      pw[0] = d2;
    }
  }
}

template <int L, typename T, int DIG = gl::kXDig>
__device__ __forceinline__ void split_column(const T (&v)[L], const Scale& s, uint32_t (&w)[L / 16][DIG][4]) {
  // w[seg][plane][word]
#pragma unroll
  for (int seg = 0; seg < L / 16; ++seg)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      long long xi[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) xi[e] = fixed_of(v[16 * seg + 4 * q + e], s);
      uint32_t pw[DIG];
      planes4d<DIG>(xi, pw);
#pragma unroll
      for (int pl = 0; pl < DIG; ++pl) w[seg][pl][q] = pw[pl];
    }
}

template <int L, typename T>
__device__ __forceinline__ float column_max(const T (&v)[L]) {
  float m = 0.f;
#pragma unroll
  for (int e = 0; e < L; ++e) m = fmaxf(m, (float)fabs((double)v[e]));
  return m;
}

template <typename T1, typename T2, int MINB>
__global__ void __launch_bounds__(kSplitThreads, MINB)
split_planes(int64_t n, int c1, const T1* __restrict__ X1, int64_t ld1, int c2, const T2* __restrict__ X2,
             int64_t ld2, int NP, bool vec1, bool vec2, uint8_t* __restrict__ planes, int* __restrict__ exps,
             bool slow) {
  // Two passes over the CTA's chunk x column pair, kSplitSeg segments of 16
  // rows per thread: the max pass reads with normal caching so that the
  // encode pass re-reads from L2; the encode pass converts both columns of
  // a segment together so each plane store fills a whole 32-byte sector.
  // Few registers live per thread -> several CTAs per SM.
  __shared__ float red[2][kSplitThreads / 32];
  const int c = blockIdx.x;
  const int j0 = 2 * blockIdx.y;
  // values are held as binary32 when both inputs are binary32 (exact), else
  // as binary64 (binary32 embeds exactly)
  using TV = typename std::conditional<sizeof(T1) == 4 && sizeof(T2) == 4, float, double>::type;
  auto load = [&](int h, int64_t base, TV (&v)[16], auto pol) {
    constexpr int P = decltype(pol)::value;
    const int j = j0 + h;
    if (j < c1) loadL<16, T1, TV, P>(X1 + (int64_t)j * ld1, base, n, vec1, v);
    else if (j < c1 + c2) loadL<16, T2, TV, P>(X2 + (int64_t)(j - c1) * ld2, base, n, vec2, v);
    else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = TV(0);  // UMMA N padding
    }
  };
  using keep = std::integral_constant<int, 1>;
  using last = std::integral_constant<int, 2>;
  auto row0 = [&](int sg) { return (int64_t)c * kChunk + (int64_t)sg * (16 * kSplitThreads) + 16 * threadIdx.x; };
  float mx[2] = {0.f, 0.f};
#pragma unroll 2
  for (int sg = 0; sg < kSplitSeg; ++sg) {
    TV v[2][16];
    load(0, row0(sg), v[0], keep{});
    load(1, row0(sg), v[1], keep{});
    mx[0] = fmaxf(mx[0], column_max(v[0]));
    mx[1] = fmaxf(mx[1], column_max(v[1]));
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
    for (int o = 16; o; o >>= 1) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], o));
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = mx[0];
    red[1][threadIdx.x >> 5] = mx[1];
  }
  __syncthreads();
  Scale sc[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    float m = 0.f;
#pragma unroll
    for (int q = 0; q < kSplitThreads / 32; ++q) m = fmaxf(m, red[h][q]);
    int E = 0;
    if (m > 0.f) frexpf(m, &E);  // m < 2^E; float rounding is monotone, so every |x| < 2^E
    if (threadIdx.x == 0) exps[(int64_t)c * NP + j0 + h] = E;
    sc[h].s = ldexp(1.0, 46 - E);
    sc[h].fast = 46 - E >= -126 && 46 - E <= 127 && !slow;
    sc[h].sf = sc[h].fast ? (float)sc[h].s : 1.f;
  }
  // encode pass, software-pipelined: segment sg + 1 is in flight while sg
  // is converted and stored
  TV v[2][16], vn[2][16];
  load(0, row0(0), vn[0], last{});
  load(1, row0(0), vn[1], last{});
#pragma unroll 1
  for (int sg = 0; sg < kSplitSeg; ++sg) {
    const int64_t base = row0(sg);
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 16; ++e) v[h][e] = vn[h][e];
    if (sg + 1 < kSplitSeg) {
      load(0, row0(sg + 1), vn[0], last{});
      load(1, row0(sg + 1), vn[1], last{});
    }
    uint32_t w[2][1][gl::kXDig][4];  // [column][seg][plane][word]
    split_column(v[0], sc[0], w[0]);
    split_column(v[1], sc[1], w[1]);
#pragma unroll
    for (int pl = 0; pl < gl::kXDig; ++pl) {
      uint4* dst = reinterpret_cast<uint4*>(planes + gl::x_offset(pl, j0, base, NP));
      __stcs(dst, make_uint4(w[0][0][pl][0], w[0][0][pl][1], w[0][0][pl][2], w[0][0][pl][3]));
      __stcs(dst + 1, make_uint4(w[1][0][pl][0], w[1][0][pl][1], w[1][0][pl][2], w[1][0][pl][3]));
    }
  }
}

// ---- pre-pass as two streaming kernels (default) ---------------------------------
// chunk_max: grid (nchunks, NP), one CTA per (chunk, column): every thread
// keeps 16 vector loads in flight, then a CTA max -> the chunk exponent E.
// encode: one thread per (16-row segment, column pair), no barrier and few
// registers, so many segments are in flight per SM; it converts exactly as
// split_planes does (same exponents, same integers, same plane bytes).
template <typename T1, typename T2>
__device__ __forceinline__ const void* col_ptr(int j, int c1, const T1* X1, int64_t ld1, int c2, const T2* X2,
                                               int64_t ld2) {
  if (j < c1) return X1 + (int64_t)j * ld1;
  if (j < c1 + c2) return X2 + (int64_t)(j - c1) * ld2;
  return nullptr;
}

template <typename T1, typename T2>
__global__ void __launch_bounds__(256)
chunk_max(int64_t n, int c1, const T1* __restrict__ X1, int64_t ld1, int c2, const T2* __restrict__ X2, int64_t ld2,
          int NP, bool vec1, bool vec2, int* __restrict__ exps) {
  __shared__ float red[8];
  const int c = blockIdx.x, j = blockIdx.y;
  const int64_t r0 = (int64_t)c * kChunk;
  float m = 0.f;
  if (j < c1 + c2) {
    const bool one = j < c1;
    const bool vec = one ? vec1 : vec2;
    if (one && sizeof(T1) == 4 && vec && r0 + kChunk <= n) {
      const float4* p = reinterpret_cast<const float4*>(X1 + (int64_t)j * ld1 + r0);
      float4 f[kChunk / 4 / 256];
#pragma unroll
      for (int i = 0; i < kChunk / 4 / 256; ++i) f[i] = __ldg(p + threadIdx.x + 256 * i);
#pragma unroll
      for (int i = 0; i < kChunk / 4 / 256; ++i)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(f[i].x), fabsf(f[i].y)), fmaxf(fabsf(f[i].z), fabsf(f[i].w))));
    } else if (!one && sizeof(T2) == 4 && vec && r0 + kChunk <= n) {
      const float4* p = reinterpret_cast<const float4*>(X2 + (int64_t)(j - c1) * ld2 + r0);
      float4 f[kChunk / 4 / 256];
#pragma unroll
      for (int i = 0; i < kChunk / 4 / 256; ++i) f[i] = __ldg(p + threadIdx.x + 256 * i);
#pragma unroll
      for (int i = 0; i < kChunk / 4 / 256; ++i)
        m = fmaxf(m, fmaxf(fmaxf(fabsf(f[i].x), fabsf(f[i].y)), fmaxf(fabsf(f[i].z), fabsf(f[i].w))));
    } else {
      const int64_t r1 = min(n, r0 + kChunk);
      for (int64_t r = r0 + threadIdx.x; r < r1; r += 256) {
        const double v = one ? (double)X1[(int64_t)j * ld1 + r] : (double)X2[(int64_t)(j - c1) * ld2 + r];
        m = fmaxf(m, (float)fabs(v));
      }
    }
  }
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) mm = fmaxf(mm, red[q]);
    int E = 0;
    if (mm > 0.f) frexpf(mm, &E);  // mm < 2^E; float rounding is monotone, so every |x| < 2^E
    exps[(int64_t)c * NP + j] = E;
  }
}

template <typename T1, typename T2, int DIG>
__global__ void __launch_bounds__(256, 4)
encode_planes(int64_t n, int c1, const T1* __restrict__ X1, int64_t ld1, int c2, const T2* __restrict__ X2,
              int64_t ld2, int NP, bool vec1, bool vec2, int64_t nseg, const int* __restrict__ exps,
              uint8_t* __restrict__ planes) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nseg * (NP / 2)) return;
  // column pairs fastest: the pairs of one segment write each plane's
  // NG x 16-byte run of the tile contiguously (whole lines per warp)
  const int64_t seg = idx / (NP / 2);
  const int j0 = 2 * (int)(idx % (NP / 2));
  const int64_t base = seg * 16;
  const int64_t chunk = base / kChunk;
  using TV = typename std::conditional<sizeof(T1) == 4 && sizeof(T2) == 4, float, double>::type;
  TV v[2][16];
  Scale sc[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = j0 + h;
    if (j < c1) loadL<16, T1, TV>(X1 + (int64_t)j * ld1, base, n, vec1, v[h]);
    else if (j < c1 + c2) loadL<16, T2, TV>(X2 + (int64_t)(j - c1) * ld2, base, n, vec2, v[h]);
    else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[h][e] = TV(0);  // UMMA N padding
    }
    const int E = __ldg(exps + chunk * NP + j);
    constexpr int kBits = 8 * DIG - 2;
    sc[h].s = ldexp(1.0, kBits - E);
    sc[h].fast = kBits - E >= -126 && kBits - E <= 127;
    sc[h].sf = sc[h].fast ? (float)sc[h].s : 1.f;
  }
  uint32_t w[2][1][DIG][4];  // [column][seg][plane][word]
  split_column<16, TV, DIG>(v[0], sc[0], w[0]);
  split_column<16, TV, DIG>(v[1], sc[1], w[1]);
#pragma unroll
  for (int pl = 0; pl < DIG; ++pl) {
    uint4* dst = reinterpret_cast<uint4*>(planes + gl::x_offset(pl, j0, base, NP, DIG));
    __stcs(dst, make_uint4(w[0][0][pl][0], w[0][0][pl][1], w[0][0][pl][2], w[0][0][pl][3]));
    __stcs(dst + 1, make_uint4(w[1][0][pl][0], w[1][0][pl][1], w[1][0][pl][2], w[1][0][pl][3]));
  }
}

// encode_tile (default): one CTA per 128-row K tile.  A warp reads 128 rows
// of one column as ONE coalesced 512-byte run (lane L: rows 4 L .. 4 L + 3)
// -- encode_planes' thread-per-(16 rows, column pair) mapping made every
// warp load touch 32 lines 64 MB apart at the C5 shape (ncu: lg_throttle,
// 2.8 TB/s) -- converts its four entries per column into one 32-bit word
// per plane, stages the tile in shared memory in the operand layout (rows
// of a K chunk padded by 16 bytes: conflict-free) and the CTA writes the
// tile's DIG x 128 x NP bytes, contiguous in HBM, as whole lines.  Same
// exponents, integers and plane bytes as encode_planes.
template <typename T1, typename T2, int DIG>
__global__ void __launch_bounds__(256, 4)
encode_tile(int64_t n, int c1, const T1* __restrict__ X1, int64_t ld1, int c2, const T2* __restrict__ X2,
            int64_t ld2, int NP, bool vec1, bool vec2, const int* __restrict__ exps, uint8_t* __restrict__ planes) {
  extern __shared__ __align__(16) uint32_t enc_sm[];
  using TV = typename std::conditional<sizeof(T1) == 4 && sizeof(T2) == 4, float, double>::type;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blockIdx.x * kBK;
  const int64_t chunk = base / kChunk;
  const int NG = gl::np_group(NP, DIG);
  const int rowW = DIG * NP * 4;   // words per K chunk (16 rows) of the tile
  const int S = rowW + 4;          // padded: the 8 K chunks of a warp store hit distinct banks
  const int kc = lane >> 2, b4 = lane & 3;
  constexpr int kMaxCols = 8;      // NP / 8 columns per warp, NP <= 64
  TV v[kMaxCols][4];
  const int ncw = NP / 8;
  const int64_t r0 = base + 4 * lane;
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) {
    if (i >= ncw) break;
    const int j = warp + 8 * i;
#pragma unroll
    for (int e = 0; e < 4; ++e) v[i][e] = TV(0);
    if (j < c1) loadL<4, T1, TV>(X1 + (int64_t)j * ld1, r0, n, vec1, v[i]);
    else if (j < c1 + c2) loadL<4, T2, TV>(X2 + (int64_t)(j - c1) * ld2, r0, n, vec2, v[i]);
  }
#pragma unroll
  for (int i = 0; i < kMaxCols; ++i) {
    if (i >= ncw) break;
    const int j = warp + 8 * i;
    const int E = __ldg(exps + chunk * NP + j);
    constexpr int kBits = 8 * DIG - 2;
    Scale sc;
    sc.s = ldexp(1.0, kBits - E);
    sc.fast = kBits - E >= -126 && kBits - E <= 127;
    sc.sf = sc.fast ? (float)sc.s : 1.f;
    long long xi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) xi[e] = fixed_of(v[i][e], sc);
    uint32_t pw[DIG];
    planes4d<DIG>(xi, pw);
    const int g = j / NG, jj = j % NG;
#pragma unroll
    for (int pl = 0; pl < DIG; ++pl) enc_sm[kc * S + ((g * DIG + pl) * NG + jj) * 4 + b4] = pw[pl];
  }
  __syncthreads();
  const int nq = (kBK / 16) * DIG * NP;  // 16-byte words of the tile
  uint4* dst = reinterpret_cast<uint4*>(planes + (int64_t)blockIdx.x * ((int64_t)DIG * kBK * NP));
  for (int q = threadIdx.x; q < nq; q += 256) {
    const int kq = q / (DIG * NP), rem = q % (DIG * NP);
    __stcs(dst + q, *reinterpret_cast<const uint4*>(&enc_sm[kq * S + rem * 4]));
  }
}

template <int NP, int ST, int DIG = gl::kXDig>
struct Smem {
  static constexpr int S = ST;
  uint8_t a[S][2][kBK / 16][kTM][16];  // one q tile
  uint8_t b[S][kBK / 16][DIG * NP][16];  // one X-plane tile: [kc][group, plane, col][16]
  uint64_t full[S], empty[S];
  uint64_t tfull[2], tempty[2];
  uint32_t tbase;
};

// LEAN: 192 threads (producer warp 0, MMA warp 1, epilogue warps 2..5 on TMEM
// lane quadrants warp & 3), <= 168 registers, two stages -- sized to share
// an SM with one CTA of the staged projection, so the sketch of the NEXT
// block's W runs on the tensor pipe while the projection keeps the FP32
// pipe busy (the sweep issues them on two streams).
template <int NP, int ST, bool LEAN, int DIG = gl::kXDig>
__device__ __forceinline__ void
gauss_tc_body(int64_t n, int ncols, const uint8_t* __restrict__ qt, int64_t ldt, int k,
              const uint8_t* __restrict__ planes1, const int* __restrict__ exps1, int tiles_per_cta,
              double* __restrict__ ws1, int dbg, int pairs, int ncols2, const uint8_t* __restrict__ planes2,
              const int* __restrict__ exps2, double* __restrict__ ws2, int qpl = 2) {
  // qpl == 1: the table's lo plane is zero (8-bit operator): only the hi plane
  // is copied and multiplied (TMEM block DIG stays as the epilogue zeroed it).
  // pairs == 2: CTAs 2 mt and 2 mt + 1 own the same 128 sketch rows and K
  // range for two inputs (two column halves of > 64 columns that do not fit
  // one CTA's TMEM); launched side by side they read each q tile once from
  // HBM and once from L2.
  const int half = pairs == 2 ? (int)(blockIdx.x & 1) : 0;
  const uint8_t* __restrict__ planes = half ? planes2 : planes1;
  const int* __restrict__ exps = half ? exps2 : exps1;
  double* __restrict__ ws = half ? ws2 : ws1;
  if (half) ncols = ncols2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  Smem<NP, ST, DIG>& S = *reinterpret_cast<Smem<NP, ST, DIG>*>(smem_raw);
  constexpr int kStages = ST;
  constexpr int kDig = DIG, kBlk = kDig + 1;  // digit planes, TMEM weight blocks
  constexpr int kGroupCols = kBlk * NP;
  constexpr int kBufs = (2 * kGroupCols <= 512) ? 2 : 1;
  constexpr uint32_t kAlloc = kBufs * kGroupCols <= 64 ? 64 : kBufs * kGroupCols <= 128 ? 128
                              : kBufs * kGroupCols <= 256 ? 256 : 512;
  static_assert(kGroupCols <= 512, "TMEM: 7 weight blocks x NP columns must fit 512");
  constexpr uint32_t kABytes = 2 * kTM * kBK, kBBytes = kDig * kBK * NP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x / pairs;
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
        const uint32_t abytes = qpl == 1 ? kABytes / 2 : kABytes;  // the hi plane comes first in a tile
        tc::mbar_arrive_expect_tx(&S.full[s], abytes + kBBytes);
        tc::bulk_g2s(&S.a[s][0][0][0][0], qtile + kt * 2 * gl::kTileBytes, abytes, &S.full[s]);
        tc::bulk_g2s(&S.b[s][0][0][0], planes + kt * (int64_t)kBBytes, kBBytes, &S.full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      // Per K step and column group g: two MMAs share the B operand
      // [b5 | .. | b0] (N = 6 NG, all s8).  qh x B lands on TMEM blocks
      // 0..5 of the group, ql x B on blocks 1..6 (D shifted by NG columns),
      // so block w accumulates exactly the products of weight 2^(48 - 8w).  The accumulators are zeroed by the epilogue, every MMA
      // accumulates.
      constexpr int NG = gl::np_group(NP, DIG);
      constexpr int NGRP = NP / NG;
      static_assert((kDig * NG) % 16 == 0 && kDig * NG <= 256 && NP % NG == 0, "UMMA N (M = 128)");
      constexpr uint32_t ID_HI = tc::idesc_i8(kTM, kDig * NG, true, true);
      constexpr uint32_t ID_LO = tc::idesc_i8(kTM, kDig * NG, false, true);
      int seg_i = 0;
      for (int t = 0; t < T; ++t) {
        const int s = t % kStages;
        const int64_t kt = kt_beg + t;
        const bool seg_first = (t == 0) || (kt % kTPC == 0);
        const bool seg_last = (t == T - 1) || ((kt + 1) % kTPC == 0);
        const int buf = seg_i % kBufs;
        if (seg_first) tc::mbar_wait(&S.tempty[buf], (seg_i / kBufs) & 1);
        tc::mbar_wait(&S.full[s], (t / kStages) & 1);
        tc::tc_fence_after();
        const uint32_t d = tbase + buf * kGroupCols;
        if (!(dbg & 1)) {
#pragma unroll
          for (int ks = 0; ks < kBK / 32; ++ks) {
            const uint64_t ah = tc::sdesc_kmajor(tc::smem_u32(&S.a[s][0][2 * ks][0][0]), kTM * 16, 128);
            const uint64_t al = tc::sdesc_kmajor(tc::smem_u32(&S.a[s][1][2 * ks][0][0]), kTM * 16, 128);
#pragma unroll
            for (int g = 0; g < NGRP; ++g) {
              const uint64_t b = tc::sdesc_kmajor(tc::smem_u32(&S.b[s][2 * ks][0][0]) + g * (kDig * NG * 16),
                                                  kDig * NP * 16, 128);
              // the first qh MMA of a segment overwrites blocks 0..5 (no
              // zeroing needed); block 6 (ql x b0 only) is zeroed by the epilogue
              tc::mma_i8(d + g * kBlk * NG, ah, b, ID_HI, (seg_first && ks == 0) ? 0u : 1u);
              if (qpl == 2) tc::mma_i8(d + g * kBlk * NG + NG, al, b, ID_LO, 1u);
            }
          }
        }
        tc::mma_commit(&S.empty[s]);
        if (seg_last) {
          tc::mma_commit(&S.tfull[buf]);
          ++seg_i;
        }
      }
    }
  } else if (LEAN ? (warp >= 2 && warp < 6) : warp >= 4) {
    // ---------------- epilogue ----------------
    constexpr int NG = gl::np_group(NP, DIG);
    static_assert(NG % 8 == 0, "epilogue drains 8 columns at a time");
    const int q = warp & 3;  // TMEM lane quadrant (warps may only touch lanes 32 (warp % 4) ..)
    const int r = mt * kTM + q * 32 + lane;
    const uint32_t lane_base = tbase + ((uint32_t)(q * 32) << 16);
    double acc[NP];  // this row's fp64 partial sketch, all columns
#pragma unroll
    for (int j = 0; j < NP; ++j) acc[j] = 0.0;
    // zero both accumulator buffers, then hand them to the MMA issuer
    for (int b = 0; b < kBufs; ++b) {
      for (int c0 = 0; c0 < kGroupCols; c0 += 8) tc::tmem_st8_zero(lane_base + b * kGroupCols + c0);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[b]);
    }
    int ci = 0;
    for (int64_t ks = kt_beg; ks < kt_end; ++ci) {
      const int64_t chunk = ks / kTPC;
      ks = min(kt_end, (chunk + 1) * kTPC);
      const int buf = ci % kBufs;
      tc::mbar_wait(&S.tfull[buf], (ci / kBufs) & 1);
      tc::tc_fence_after();
      const uint32_t la = lane_base + buf * kGroupCols;
      const int* ex = exps + chunk * NP;
      // With room for a second register copy (NP <= 40), the chunk's terms
      // are staged in t[] and TMEM is handed back before the fp64 adds.
      constexpr bool kStage = NP <= 40 && !LEAN;
      double t[kStage ? NP : 1];
#pragma unroll
      for (int c0 = 0; c0 < NP; c0 += 8) {
        const uint32_t gbase = la + (c0 / NG) * kBlk * NG + (c0 % NG);
        uint32_t g[kBlk][8];
#pragma unroll
        for (int w = 0; w < kBlk; ++w) tc::tmem_ld8(gbase + w * NG, g[w]);
        tc::tmem_ld_wait();
        if constexpr (kStage) {
          tc::tmem_st8_zero(gbase + (kBlk - 1) * NG);
        } else {  // (the stores also keep ptxas from overlapping groups: registers)
#pragma unroll
          for (int w = 0; w < kBlk; ++w) tc::tmem_st8_zero(gbase + w * NG);
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          // integer recombination of the weights 2^48, .., 2^0 in two exact
          // int64 halves (hi: 2^48 .. 2^32 -> < 2^47; lo: 2^24 .. 2^0 ->
          // < 2^55), then two binary64 roundings; the scalings by 2^(e+32)
          // and 2^e are exact (normal binary64 powers of two for every
          // binary32 / binary64 chunk exponent), i.e. equal to ldexp
          double term;
          const int e = ex[c0 + jj] - (8 * DIG - 2);
          if constexpr (DIG == gl::kXDig) {
            const long long hi = ((long long)(int)g[0][jj] << 16) + ((long long)(int)g[1][jj] << 8) +
                                 (long long)(int)g[2][jj];
            const long long lo = ((long long)(int)g[3][jj] << 24) + ((long long)(int)g[4][jj] << 16) +
                                 ((long long)(int)g[5][jj] << 8) + (long long)(int)g[6][jj];
            if constexpr (kStage) {
              const double shi = __longlong_as_double((long long)(e + 32 + 1023) << 52);
              const double slo = __longlong_as_double((long long)(e + 1023) << 52);
              term = __dadd_rn(__dmul_rn((double)hi, shi), __dmul_rn((double)lo, slo));
            } else {  // (ldexp: fewer live registers at NP = 48 / 64)
              term = ldexp((double)hi, e + 32) + ldexp((double)lo, e);
            }
          } else {
            // DIG + 1 weight blocks, < 2^30 each: the exact sum fits one int64
            // (< 2^63 at DIG = 4); one binary64 rounding
            long long v = 0;
#pragma unroll
            for (int w = 0; w < kBlk; ++w) v += (long long)(int)g[w][jj] << (8 * (kDig - w));
            term = ldexp((double)v, e);
          }
          if constexpr (kStage) t[c0 + jj] = term;
          else acc[c0 + jj] += term;
        }
      }
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&S.tempty[buf]);
      if constexpr (kStage) {
#pragma unroll
        for (int j = 0; j < NP; ++j) acc[j] += t[j];
      }
    }
    if (r < k) {
      double* dst = ws + (int64_t)blockIdx.y * k * ncols + r;
#pragma unroll
      for (int j = 0; j < NP; ++j)
        if (j < ncols) dst[(int64_t)j * k] = acc[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) tc::tmem_dealloc(tbase, kAlloc);
}

template <int NP, int ST, int DIG>
__global__ void __launch_bounds__(kThreads, 1)
gauss_tc_partial(int64_t n, int ncols, const uint8_t* __restrict__ qt, int64_t ldt, int k,
                 const uint8_t* __restrict__ planes1, const int* __restrict__ exps1, int tiles_per_cta,
                 double* __restrict__ ws1, int dbg, int pairs, int ncols2, const uint8_t* __restrict__ planes2,
                 const int* __restrict__ exps2, double* __restrict__ ws2, int qpl) {
  gauss_tc_body<NP, ST, false, DIG>(n, ncols, qt, ldt, k, planes1, exps1, tiles_per_cta, ws1, dbg, pairs, ncols2,
                                    planes2, exps2, ws2, qpl);
}

constexpr int kLeanThreads = 192;
template <int NP, int ST>
__global__ void __launch_bounds__(kLeanThreads, 2)  // (2 x 192 threads: <= 168 registers)
gauss_tc_lean(int64_t n, int ncols, const uint8_t* __restrict__ qt, int64_t ldt, int k,
              const uint8_t* __restrict__ planes1, const int* __restrict__ exps1, int tiles_per_cta,
              double* __restrict__ ws1, int dbg, int pairs, int ncols2, const uint8_t* __restrict__ planes2,
              const int* __restrict__ exps2, double* __restrict__ ws2) {
  gauss_tc_body<NP, ST, true>(n, ncols, qt, ldt, k, planes1, exps1, tiles_per_cta, ws1, dbg, pairs, ncols2, planes2,
                              exps2, ws2);
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

// padded column count (UMMA N = DIG NG must be a multiple of 16: no NP = 40 at DIG = 3)
int np_for(int ncols, int dig = gl::kXDig) {
  return ncols <= 16 ? 16 : ncols <= 32 ? 32 : (ncols <= 40 && dig != 3) ? 40 : ncols <= 48 ? 48 : 64;
}

int dbg_flag() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RB_TC_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

struct Half2 {  // the second input of a paired launch (pairs == 2)
  int pairs = 1, ncols = 0, qpl = 2;
  const uint8_t* planes = nullptr;
  const int* exps = nullptr;
};

template <int NP, int DIG = gl::kXDig>
int launch_np(int64_t n, int ncols, const uint8_t* qt, int64_t ldt, int k, const uint8_t* planes, const int* exps,
              double* part, size_t part_bytes, int* splits_out, cudaStream_t st, const Half2& h2 = Half2(),
              bool lean = false) {
  const int mt = ceil_div(k, kTM);
  // one wave: floor(SMs / m-tiles) K ranges of equal tile counts.  A paired
  // launch keeps the same K ranges (two waves of CTA pairs), so each input's
  // partials -- and the result bits -- equal those of its own launch.
  const int64_t ktn = (n + kBK - 1) / kBK;
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(ktn, sm_count() / mt));
  // a paired launch keeps each half's partials in its own half of `part`
  if (h2.pairs == 2) part_bytes = (part_bytes / 2) & ~(size_t)255;
  const size_t per = (size_t)k * std::max(ncols, h2.ncols) * sizeof(double);
  if ((size_t)splits * per > part_bytes) splits = (int)std::max<size_t>(1, part_bytes / per);
  RB_REQUIRE((size_t)splits * per <= part_bytes, "gaussian tc: workspace too small");
  const int tpc = (int)((ktn + splits - 1) / splits);
  splits = (int)((ktn + tpc - 1) / tpc);
  static int env_st = -1;
  if (env_st < 0) {
    const char* e = getenv("RB_TC_STAGES");
    env_st = e ? atoi(e) : 0;
  }
  constexpr int kMax = max_stages<NP, DIG>();
  const int st_req = env_st > 0 ? std::min(env_st, kMax) : std::min(kMax, DIG == gl::kXDig ? 3 : 4);
#define RB_GL(STG)                                                                                               \
  {                                                                                                              \
    const size_t smem = sizeof(Smem<NP, STG, DIG>) + 1024;                                                       \
    cudaFuncSetAttribute(gauss_tc_partial<NP, STG, DIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    RB_KLAUNCH gauss_tc_partial<NP, STG, DIG><<<dim3(mt * h2.pairs, splits), kThreads, smem, st>>>(              \
        n, ncols, qt, ldt, k, planes, exps, tpc, part, dbg_flag(), h2.pairs, h2.ncols, h2.planes, h2.exps,       \
        part + part_bytes / sizeof(double), h2.qpl);                                                             \
  }
  if (lean && h2.pairs == 1 && DIG == gl::kXDig) {
    // two stages: shares the SM with one projection CTA
    const size_t smem = sizeof(Smem<NP, 2>) + 1024;
    cudaFuncSetAttribute(gauss_tc_lean<NP, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(gauss_tc_lean<NP, 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    RB_KLAUNCH gauss_tc_lean<NP, 2><<<dim3(mt, splits), kLeanThreads, smem, st>>>(
        n, ncols, qt, ldt, k, planes, exps, tpc, part, dbg_flag(), 1, 0, nullptr, nullptr, nullptr);
  } else if (st_req >= 4 && kMax >= 4) RB_GL((kMax >= 4 ? 4 : 1))
  else if (st_req >= 3 && kMax >= 3) RB_GL((kMax >= 3 ? 3 : 1))
  else RB_GL(2)
#undef RB_GL
  *splits_out = splits;
  return check_launch("gauss_tc_partial");
}

bool aligned16(const void* p, int64_t ld, int esz) {
  return p && ((uintptr_t)p % 16 == 0) && ((ld * esz) % 16 == 0);
}

template <typename T1>
void launch_split(int xd2, dim3 g, int64_t n, int c1, const void* X1, int64_t ld1, int c2, const void* X2, int64_t ld2,
                  int NP, uint8_t* planes, int* exps, cudaStream_t st, int dig = gl::kXDig) {
  // RB_SPLIT_MODE=1: the single-kernel two-pass split_planes (kept for
  // measurement); default: chunk_max + encode_planes (same bytes).
  // RB_SPLIT_SLOW=1: binary64 conversion for binary32 inputs too (the
  // cross-check of the binary32 fast path -- same integers by construction)
  static int mode = -1, slow = 0;
  if (mode < 0) {
    const char* e = getenv("RB_SPLIT_MODE");
    mode = e ? atoi(e) : 3;
    const char* s = getenv("RB_SPLIT_SLOW");
    slow = s ? atoi(s) : 0;
  }
  const bool v1 = aligned16(X1, ld1, sizeof(T1));
  const int64_t nseg = (int64_t)g.x * (kChunk / 16);
#define RB_SPL(T2)                                                                                               \
  do {                                                                                                           \
    const bool v2 = aligned16(X2, ld2, sizeof(T2));                                                              \
    if ((mode == 1 || slow) && dig == gl::kXDig) {                                                               \
      RB_KLAUNCH split_planes<T1, T2, 3><<<g, kSplitThreads, 0, st>>>(n, c1, (const T1*)X1, ld1, c2,             \
                                                                      (const T2*)X2, ld2, NP, v1, v2, planes,    \
                                                                      exps, slow != 0);                          \
    } else {                                                                                                     \
      RB_KLAUNCH chunk_max<T1, T2><<<dim3(g.x, NP), 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,   \
                                                                  ld2, NP, v1, v2, exps);                        \
      const unsigned eg = (unsigned)ceil_div(nseg * (NP / 2), 256);                                              \
      const unsigned tg = (unsigned)(nseg * 16 / kBK);                                                           \
      const size_t tsm = (size_t)(kBK / 16) * ((size_t)dig * NP * 4 + 4) * 4;                                     \
      if (mode == 3) {                                                                                           \
        if (dig == 3) {                                                                                          \
          cudaFuncSetAttribute(encode_tile<T1, T2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);   \
          RB_KLAUNCH encode_tile<T1, T2, 3><<<tg, 256, tsm, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,  \
                                                                  ld2, NP, v1, v2, exps, planes);                \
        } else if (dig == 4) {                                                                                   \
          cudaFuncSetAttribute(encode_tile<T1, T2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);   \
          RB_KLAUNCH encode_tile<T1, T2, 4><<<tg, 256, tsm, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,  \
                                                                  ld2, NP, v1, v2, exps, planes);                \
        } else {                                                                                                 \
          cudaFuncSetAttribute(encode_tile<T1, T2, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);   \
          RB_KLAUNCH encode_tile<T1, T2, 6><<<tg, 256, tsm, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,  \
                                                                  ld2, NP, v1, v2, exps, planes);                \
        }                                                                                                        \
      } else if (dig == 3) {                                                                                     \
        RB_KLAUNCH encode_planes<T1, T2, 3><<<eg, 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,    \
                                                                ld2, NP, v1, v2, nseg, exps, planes);            \
      } else if (dig == 4) {                                                                                     \
        RB_KLAUNCH encode_planes<T1, T2, 4><<<eg, 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,    \
                                                                ld2, NP, v1, v2, nseg, exps, planes);            \
      } else {                                                                                                   \
        RB_KLAUNCH encode_planes<T1, T2, 6><<<eg, 256, 0, st>>>(n, c1, (const T1*)X1, ld1, c2, (const T2*)X2,    \
                                                                ld2, NP, v1, v2, nseg, exps, planes);            \
      }                                                                                                          \
    }                                                                                                            \
  } while (0)
  if (xd2 == RB_F32) RB_SPL(float);
  else RB_SPL(double);
#undef RB_SPL
}

// one launch for every (NP, DIG) the sketch supports
int launch_any(int NP, int dig, int64_t n, int ncols, const uint8_t* qt, int64_t ldt, int k, const uint8_t* planes,
               const int* exps, double* part, size_t part_b, int* splits, cudaStream_t st, const Half2& h2, bool lean) {
#define RB_LA(NPV, DG) \
  return launch_np<NPV, DG>(n, ncols, qt, ldt, k, planes, exps, part, part_b, splits, st, h2, lean)
  if (dig == 3) {
    switch (NP) {
      case 16: RB_LA(16, 3);
      case 32: RB_LA(32, 3);
      case 48: RB_LA(48, 3);
      default: RB_LA(64, 3);
    }
  }
  if (dig == 4) {
    switch (NP) {
      case 16: RB_LA(16, 4);
      case 32: RB_LA(32, 4);
      case 40: RB_LA(40, 4);
      case 48: RB_LA(48, 4);
      default: RB_LA(64, 4);
    }
  }
  switch (NP) {
    case 16: RB_LA(16, 6);
    case 32: RB_LA(32, 6);
    case 40: RB_LA(40, 6);
    case 48: RB_LA(48, 6);
    default: RB_LA(64, 6);
  }
#undef RB_LA
}

// [out1 | out2] for c1 + c2 > 64 (each <= 64): the two inputs are split into
// their own plane sets and sketched by CTA pairs of one launch that share
// every q tile (one HBM read of the table per pair instead of per input).
int sketch_gaussian_tc_pair(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2,
                            int c2, int64_t n, const uint8_t* qt, int64_t ldt, int k, double scale, double* out1,
                            int64_t ldo1, double* out2, int64_t ldo2, int acc, void* ws, size_t wsb, cudaStream_t st,
                            int dig, const void* pre2 = nullptr, int qpl = 2) {
  RB_REQUIRE(c1 >= 1 && c2 >= 1 && c1 <= 64 && c2 <= 64 && k >= 1 && out1 && out2 && ldo1 >= k && ldo2 >= k,
             "rb_sketch_gaussian (tensor pair): bad args (c1 %d, c2 %d)", c1, c2);
  RB_REQUIRE(n == 0 || (X1 && ld1 >= n && X2 && ld2 >= n && qt && ldt >= n && ldt % kBK == 0),
             "rb_sketch_gaussian (tensor pair): bad X/theta (ldt %% 128 required)");
  const int NP = std::max(np_for(c1, dig), np_for(c2, dig));
  const int nchunks = (int)((n + kChunk - 1) / kChunk);
  const int64_t ktiles = (int64_t)nchunks * kTPC;
  const size_t planes_b = (size_t)ktiles * dig * kBK * NP;
  const size_t exps_b = ((size_t)NP * nchunks * sizeof(int) + 255) / 256 * 256;
  RB_REQUIRE(ws && wsb > 2 * (planes_b + exps_b) + 2048, "rb_sketch_gaussian (tensor pair): workspace too small");
  uint8_t* pl1 = (uint8_t*)ws;
  int* ex1 = (int*)(pl1 + planes_b);
  uint8_t* pl2 = pl1 + planes_b + exps_b;
  int* ex2 = (int*)(pl2 + planes_b);
  double* part = (double*)(pl2 + planes_b + exps_b);
  if (pre2) {  // the second input's planes and exponents, encoded earlier (rb_gauss_prepass)
    pl2 = (uint8_t*)const_cast<void*>(pre2);
    ex2 = (int*)(pl2 + planes_b);
  }
  const size_t part_b = wsb - 2 * (planes_b + exps_b);
  int splits = 0;
  if (n > 0) {
    dim3 g(nchunks, NP / 2);
    if (xd1 == RB_F32) launch_split<float>(RB_F32, g, n, c1, X1, ld1, 0, nullptr, 0, NP, pl1, ex1, st, dig);
    else launch_split<double>(RB_F32, g, n, c1, X1, ld1, 0, nullptr, 0, NP, pl1, ex1, st, dig);
    if (pre2) {
    } else if (xd2 == RB_F32) launch_split<float>(RB_F32, g, n, c2, X2, ld2, 0, nullptr, 0, NP, pl2, ex2, st, dig);
    else launch_split<double>(RB_F32, g, n, c2, X2, ld2, 0, nullptr, 0, NP, pl2, ex2, st, dig);
    Half2 h2;
    h2.pairs = 2;
    h2.ncols = c2;
    h2.planes = pl2;
    h2.exps = ex2;
    h2.qpl = qpl;
    const int rc = launch_any(NP, dig, n, c1, qt, ldt, k, pl1, ex1, part, part_b, &splits, st, h2, false);
    if (rc != RB_OK) return rc;
  }
  const size_t half_b = (part_b / 2) & ~(size_t)255;
  double* part2 = part + half_b / sizeof(double);
  RB_KLAUNCH reduce_splits_tc<<<ceil_div((int64_t)k * c1, 256), 256, 0, st>>>(part, splits, k, c1, c1, scale, out1,
                                                                             ldo1, nullptr, 0, acc);
  RB_KLAUNCH reduce_splits_tc<<<ceil_div((int64_t)k * c2, 256), 256, 0, st>>>(part2, splits, k, c2, c2, scale, out2,
                                                                             ldo2, nullptr, 0, acc);
  return check_launch("rb_sketch_gaussian (tensor pair)");
}

}  // namespace

// The pre-pass of ONE input of a paired sketch on its own (planes, then
// exponents, in `out`): the sweep encodes W_(i+1) on a side stream while
// block i's projection runs, and hands the buffer to the paired call.
size_t gauss_prepass_bytes(int64_t n, int c, int c_partner, int dig) {
  const int NP = std::max(np_for(c, dig), np_for(c_partner, dig));
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  return (size_t)nchunks * kTPC * dig * kBK * NP + ((size_t)NP * nchunks * sizeof(int) + 255) / 256 * 256;
}

int gauss_prepass(int xd, const void* X, int64_t ld, int c, int c_partner, int64_t n, int dig, void* out, size_t outb,
                  cudaStream_t st) {
  RB_REQUIRE(c >= 1 && c <= 64 && c_partner >= 1 && c_partner <= 64 && n >= 1 && X && ld >= n && out &&
                 (dig == 6 || dig == 4 || dig == 3) && outb >= gauss_prepass_bytes(n, c, c_partner, dig) &&
                 (uintptr_t)out % 256 == 0,
             "rb_gauss_prepass: bad args");
  const int NP = std::max(np_for(c, dig), np_for(c_partner, dig));
  const int nchunks = (int)((n + kChunk - 1) / kChunk);
  const size_t planes_b = (size_t)nchunks * kTPC * dig * kBK * NP;
  uint8_t* pl = (uint8_t*)out;
  int* ex = (int*)(pl + planes_b);
  dim3 g(nchunks, NP / 2);
  if (xd == RB_F32) launch_split<float>(RB_F32, g, n, c, X, ld, 0, nullptr, 0, NP, pl, ex, st, dig);
  else launch_split<double>(RB_F32, g, n, c, X, ld, 0, nullptr, 0, NP, pl, ex, st, dig);
  return check_launch("rb_gauss_prepass");
}

size_t gauss_tc_ws_bytes(int64_t n, int ncols, int k) {
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  // room for a fused two-input call: <= 64 columns in one CTA, else two
  // paired halves of <= 64 columns each
  const int cols = ncols <= 64 ? 64 : 128;
  const size_t planes = (size_t)gl::kXDig * cols * nchunks * kChunk;
  const size_t exps = ((size_t)cols * nchunks * sizeof(int) + 255) / 256 * 256;
  const size_t part = (size_t)(sm_count() + 1) * std::max(k, 64) * cols * sizeof(double);
  return planes + exps + part + 1024;
}

// [out1 | out2] = scale * (q @ [X1 | X2]) on the tensor pipe; each X is
// binary32 or binary64 (n rows); c2 may be 0.
int sketch_gaussian_tc(int xd1, const void* X1, int64_t ld1, int c1, int xd2, const void* X2, int64_t ld2, int c2,
                       int64_t n, const uint8_t* qt, int64_t ldt, int k, double scale, double* out1, int64_t ldo1,
                       double* out2, int64_t ldo2, int acc, void* ws, size_t wsb, cudaStream_t st, bool lean, int dig,
                       const void* pre2, int qpl) {
  const int ncols = c1 + c2;
  RB_REQUIRE(dig == 6 || dig == 4 || dig == 3, "rb_sketch_gaussian (tensor): digits must be 6, 4 or 3 (got %d)", dig);
  RB_REQUIRE(!pre2 || ncols > 64, "rb_sketch_gaussian (tensor): a pre-encoded second input needs the paired form");
  if (ncols > 64)
    return sketch_gaussian_tc_pair(xd1, X1, ld1, c1, xd2, X2, ld2, c2, n, qt, ldt, k, scale, out1, ldo1, out2, ldo2,
                                   acc, ws, wsb, st, dig, pre2, qpl);
  RB_REQUIRE(c1 >= 1 && c2 >= 0 && ncols <= 64 && k >= 1 && ldo1 >= k && out1 && (c2 == 0 || (out2 && ldo2 >= k)),
             "rb_sketch_gaussian (tensor): bad args (c1 %d, c2 %d)", c1, c2);
  RB_REQUIRE(n == 0 || (X1 && ld1 >= n && (c2 == 0 || (X2 && ld2 >= n)) && qt && ldt >= n && ldt % kBK == 0),
             "rb_sketch_gaussian (tensor): bad X/theta (ldt %% 128 required)");
  const int NP = np_for(ncols, dig);
  const int nchunks = (int)((n + kChunk - 1) / kChunk);
  const int64_t ktiles = (int64_t)nchunks * kTPC;
  const size_t planes_b = (size_t)ktiles * dig * kBK * NP;
  const size_t exps_b = ((size_t)NP * nchunks * sizeof(int) + 255) / 256 * 256;
  RB_REQUIRE(ws && wsb > planes_b + exps_b + 1024, "rb_sketch_gaussian (tensor): workspace too small");
  uint8_t* planes = (uint8_t*)ws;
  int* exps = (int*)((uint8_t*)ws + planes_b);
  double* part = (double*)((uint8_t*)ws + planes_b + exps_b);
  const size_t part_b = wsb - planes_b - exps_b;
  int splits = 0;
  if (n > 0) {
    dim3 g(nchunks, NP / 2);
    if (xd1 == RB_F32) launch_split<float>(xd2, g, n, c1, X1, ld1, c2, X2, ld2, NP, planes, exps, st, dig);
    else launch_split<double>(xd2, g, n, c1, X1, ld1, c2, X2, ld2, NP, planes, exps, st, dig);
    Half2 h1;
    h1.qpl = qpl;
    const int rc = launch_any(NP, dig, n, ncols, qt, ldt, k, planes, exps, part, part_b, &splits, st, h1, lean);
    if (rc != RB_OK) return rc;
  }
  const int64_t tot = (int64_t)k * ncols;
  RB_KLAUNCH reduce_splits_tc<<<ceil_div(tot, 256), 256, 0, st>>>(part, splits, k, c1, ncols, scale, out1, ldo1, out2,
                                                                  ldo2, acc);
  return check_launch("rb_sketch_gaussian (tensor)");
}

}  // namespace rb
