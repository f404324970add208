// Small upper-triangular R (p <= 64) in the CONSTANT bank for the tall
// right solves X = B R^{-1} (rbgs.py:281-283 -> kernels.py:250-270).
//
// A row solve reads every R_lj once per row; from shared memory each read is
// a broadcast LDS whose 8 bytes are still written back to all 32 lanes'
// registers, and that writeback (not the DFMA pipe) bounded the kernel
// (ncu: LSU writeback ~50%, FP64 pipe ~22%).  Served from the constant bank
// the operand arrives through the uniform datapath instead: measured
// 1.06 vs 1.96 ms at 2^24 x 32 and 6.6 vs 8.5 ms at 2^24 x 64
// (tools/trsm_bench.cu, profiles/r01_trsm_variants.json), bit-identical.
//
// Each translation unit that includes this header gets its own copy (the
// anonymous namespace); load_tri_const() refreshes THIS unit's copy,
// stream-ordered: a pack kernel into a per-device staging array (a device
// global, so no allocation -- legal inside graph capture), then one
// device-to-symbol copy.  The bank is per device, not per stream, so a solve
// issued on another stream than the previous one first waits (event) for
// the previous stream's consumer kernel: two streams' solves on one device
// are serialised, never interleaved (tri_const_done() records that event).
// Inside a stream capture the cross-stream wait is not recorded; a captured
// graph must not replay concurrently with other streams' solves on its
// device (include/rbgs_b200.h, conventions).
#pragma once

#include <mutex>

#include "common.cuh"

namespace rb {
namespace {

constexpr int kTriLd = 64;
// [0, 64 * 64): R column-major, ld 64, zero padded; then 1 / R_jj (0 for j >= p)
__constant__ double c_tri[kTriLd * kTriLd + kTriLd];
__device__ double g_tri_stage[kTriLd * kTriLd + kTriLd];
#define c_tri_R c_tri
#define c_tri_inv (c_tri + kTriLd * kTriLd)

__global__ void tri_pack_kernel(int p, const double* __restrict__ R, int64_t ldr) {
  double* dst = g_tri_stage;
  for (int e = threadIdx.x; e < kTriLd * kTriLd; e += blockDim.x) {
    const int i = e % kTriLd, j = e / kTriLd;
    dst[e] = (i < p && j < p) ? R[i + (int64_t)j * ldr] : 0.0;
  }
  for (int j = threadIdx.x; j < kTriLd; j += blockDim.x)
    dst[kTriLd * kTriLd + j] = j < p ? 1.0 / R[j + (int64_t)j * ldr] : 0.0;
}

struct TriOwner {
  cudaStream_t last = nullptr;
  bool used = false;
  cudaEvent_t done = nullptr;  // recorded after the last consumer on `last`
  bool done_valid = false;
};

inline std::mutex& tri_mutex() {
  static std::mutex mu;
  return mu;
}

inline TriOwner& tri_owner(int dev) {
  static TriOwner owners[64];
  return owners[dev & 63];
}

inline bool stream_capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  return cs != cudaStreamCaptureStatusNone;
}

// Call with the tri mutex held (load_tri_const .. tri_const_done bracket one
// consumer launch).
inline int load_tri_const_locked(int p, const double* R, int64_t ldr, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  TriOwner& o = tri_owner(dev);
  if (o.used && o.last != st && o.done_valid && !stream_capturing(st))
    cudaStreamWaitEvent(st, o.done, 0);  // the previous stream's solve has read the bank
  RB_KLAUNCH tri_pack_kernel<<<1, 256, 0, st>>>(p, R, ldr);
  void* stage = nullptr;
  cudaGetSymbolAddress(&stage, g_tri_stage);
  cudaMemcpyToSymbolAsync(c_tri, stage, (kTriLd * kTriLd + kTriLd) * sizeof(double), 0,
                          cudaMemcpyDeviceToDevice, st);
  return check_launch("tri_const load");
}

inline void tri_const_done_locked(cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  TriOwner& o = tri_owner(dev);
  o.last = st;
  o.used = true;
  if (stream_capturing(st)) {
    o.done_valid = false;
    return;
  }
  if (!o.done) cudaEventCreateWithFlags(&o.done, cudaEventDisableTiming);
  o.done_valid = o.done && cudaEventRecord(o.done, st) == cudaSuccess;
}

// One row: x (registers, PB >= p columns) <- x R^{-1}, dot form, l ascending
// (shared by trsm_right_kernel and the fused projection prologue).
template <int PB, int CH = 2>
__device__ __forceinline__ void tri_solve_row(double (&x)[PB], int p) {
  // CH columns at a time as independent FMA chains (the runtime `j < p`
  // guard otherwise keeps ptxas from interleaving across columns, leaving
  // one dependent DFMA chain per thread; the standalone TRSM uses CH = 4 up
  // to 40 columns, the register-tight fused projection prologue CH = 1).  Each chain keeps its own order: l
  // ascending over the finished columns, then the group's earlier columns
  // in ascending order once they are final -- the one-column roundings.
#pragma unroll
  for (int j = 0; j < PB; j += CH) {
    if (j + CH <= PB && j + CH <= p) {
      double s[CH];
#pragma unroll
      for (int c = 0; c < CH; ++c) s[c] = x[j + c];
#pragma unroll
      for (int l = 0; l < j; ++l)
#pragma unroll
        for (int c = 0; c < CH; ++c) s[c] = fma(-x[l], c_tri_R[l + (j + c) * kTriLd], s[c]);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        x[j + c] = s[c] * c_tri_inv[j + c];
#pragma unroll
        for (int c2 = c + 1; c2 < CH; ++c2) s[c2] = fma(-x[j + c], c_tri_R[j + c + (j + c2) * kTriLd], s[c2]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int jj = j + c;
        if (jj < PB && jj < p) {
          double t = x[jj];
#pragma unroll
          for (int l = 0; l < jj; ++l) t = fma(-x[l], c_tri_R[l + jj * kTriLd], t);
          x[jj] = t * c_tri_inv[jj];
        }
      }
    }
  }
}

}  // namespace
}  // namespace rb
