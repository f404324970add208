// Layout of the gaussian table q (and of the X byte planes) in HBM, tiled for
// the tensor-core sketch: every (128 sketch rows x 128 W-rows) tile of the
// two byte planes of q is one contiguous 32 KB block, laid out exactly as the
// UMMA K-major no-swizzle operand wants it in shared memory
// ([plane][16-byte K chunk][row][16 bytes]), so one bulk async copy moves it.
#pragma once

#include <stdint.h>

namespace rb {
namespace gl {

constexpr int kTM = 128;  // sketch rows per tile (UMMA M)
constexpr int kBK = 128;  // W-rows per tile (K bytes)
constexpr int kTileBytes = kTM * kBK;  // one plane of one tile

// q planes: plane 0 = hi (s8, q >> 8), plane 1 = lo (u8, q & 255).
// ldt = padded W-row count (multiple of kBK); KT = ldt / kBK.
__host__ __device__ __forceinline__ int64_t q_offset(int plane, int r, int64_t i, int64_t ldt) {
  const int64_t KT = ldt / kBK;
  const int mt = r / kTM, rr = r % kTM;
  const int64_t kt = i / kBK;
  const int kc = (int)((i % kBK) >> 4), b = (int)(i & 15);
  return (((int64_t)mt * KT + kt) * 2 + plane) * kTileBytes + (int64_t)kc * (kTM * 16) + rr * 16 + b;
}

__host__ __device__ __forceinline__ int64_t q_bytes(int k, int64_t ldt) {
  return (int64_t)((k + kTM - 1) / kTM) * kTM * ldt * 2;
}

// X byte planes for NP padded columns, as ONE UMMA B operand per column
// group: the NP columns are cut into groups of NG = np_group(NP) (so that
// kXDig NG <= 256, the largest MMA N, and is a multiple of 16 as M = 128
// requires), and within a K chunk the B rows are ordered
// [group][plane][column], plane 0 = b5 (weight 2^40) .. plane 5 = b0.
// A tile kt is kXDig x kBK x NP bytes, [kc][group][plane][col][16 bytes].
// Digits per X entry: DIG = 6 (46-bit fixed point, binary64-grade sketches:
// the default), 4 (30 bits) or 3 (22 bits) -- the cheaper forms for inputs
// whose R tolerates them (the caller's choice, gated by the measured oracle
// drift; the tensor-pipe work is proportional to DIG).  xi = x 2^(8 DIG - 2 - E).
constexpr int kXDig = 6;  // the largest digit count (workspace sizing)
__host__ __device__ constexpr int np_group(int NP, int DIG = kXDig) {
  return DIG == 6 ? (NP <= 40 ? NP : NP == 48 ? 24 : 32) : NP;  // DIG NG <= 256, % 16 == 0
}

__host__ __device__ __forceinline__ int64_t x_offset(int plane, int j, int64_t i, int NP, int DIG = kXDig) {
  const int64_t kt = i / kBK;
  const int kc = (int)((i % kBK) >> 4), b = (int)(i & 15);
  const int NG = np_group(NP, DIG);
  const int g = j / NG, jj = j % NG;
  return kt * (DIG * (int64_t)kBK * NP) + (int64_t)kc * (DIG * NP * 16) +
         (int64_t)((g * DIG + plane) * NG + jj) * 16 + b;
}

}  // namespace gl
}  // namespace rb
