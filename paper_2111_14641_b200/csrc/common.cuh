// Shared helpers for the rbgs_b200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "../../include/rbgs_b200.h"

namespace rb {

// ---- error plumbing (host) -------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define RB_REQUIRE(cond, ...)          \
  do {                                 \
    if (!(cond)) {                     \
      ::rb::set_error(__VA_ARGS__);    \
      return RB_EINVAL;                \
    }                                  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Every kernel launch of the library goes through RB_KLAUNCH, which bumps a
// process-wide counter (rb_launch_count) -- the bench's "gpu_launches".
extern unsigned long long g_launches;
#define RB_KLAUNCH ::rb::g_launches++,

int sm_count();

constexpr int kWarp = 32;

// ---- typed loads -------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double ld_f64(const T* p) { return static_cast<double>(*p); }

template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) { return __ldcs(p); }

// ---- reductions ----------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of one double per thread; result valid in thread 0.
// `red` must hold blockDim.x / 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

// ---- Philox4x32-10 (Salmon et al. SC'11); oracle/philox.py is the CPU twin --
struct u32x4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ u32x4 philox4x32_10(u32x4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    c = u32x4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

constexpr uint32_t kTagGauss = 0x47415553u;   // 'GAUS'
constexpr uint32_t kTagSparse = 0x53505253u;  // 'SPRS'

// Sparse-sign column of global W-row i: the s distinct rows and signs
// (+1/-1) drawn from the Philox word stream, duplicates skipped
// (oracle/sketches.py::sparse_sign_rows).  s <= 16.
__device__ __forceinline__ int sparse_sign_column(uint64_t i, uint64_t seed, int k, int s,
                                                  int* rows, int* sgn) {
  int have = 0;
  for (uint32_t t = 0; have < s; ++t) {
    const u32x4 w4 = philox4x32_10(u32x4{(uint32_t)i, (uint32_t)(i >> 32), t, kTagSparse},
                                   (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (have >= s) break;
      const int cand = (int)(((uint64_t)(ws[j] >> 1) * (uint64_t)k) >> 31);
      bool dup = false;
      for (int q = 0; q < have; ++q) dup |= (rows[q] == cand);
      if (!dup) {
        rows[have] = cand;
        sgn[have] = (ws[j] & 1u) ? -1 : 1;
        ++have;
      }
    }
  }
  return have;
}

// Register-resident variant (no local memory): the same rows, signs and
// order as sparse_sign_column for s <= SMAX, every array index static.
// tr[q] = (row << 1) | (negative sign).
template <int SMAX>
__device__ __forceinline__ void sparse_sign_targets(uint64_t i, uint64_t seed, int k, int s, int (&tr)[SMAX]) {
  int have = 0;
#pragma unroll
  for (int q = 0; q < SMAX; ++q) tr[q] = 0;
  for (uint32_t t = 0; have < s; ++t) {
    const u32x4 w4 = philox4x32_10(u32x4{(uint32_t)i, (uint32_t)(i >> 32), t, kTagSparse},
                                   (uint32_t)seed, (uint32_t)(seed >> 32));
    const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cand = (int)(((uint64_t)(ws[j] >> 1) * (uint64_t)k) >> 31);
      bool dup = false;
#pragma unroll
      for (int q = 0; q < SMAX; ++q) dup |= (q < have) && ((tr[q] >> 1) == cand);
      const bool take = !dup && have < s;
#pragma unroll
      for (int q = 0; q < SMAX; ++q)
        if (take && q == have) tr[q] = (cand << 1) | (int)(ws[j] & 1u);
      have += take ? 1 : 0;
    }
  }
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

}  // namespace rb
