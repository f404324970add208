#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cstring>
#include <cuda_runtime.h>
// V0: dot form (current), 1 row/thread
template <int PB>
__global__ void __launch_bounds__(256, 2) v0(int64_t n, int p, const float* B, int64_t ldb, const double* __restrict__ Rg, int64_t ldr, float* Xo, int64_t ldx) {
  constexpr int LD = (PB + 1) & ~1;
  __shared__ __align__(16) double sR[LD * PB];
  __shared__ double sInv[PB];
  for (int e = threadIdx.x; e < LD * PB; e += blockDim.x) { const int i = e % LD, j = e / LD; sR[e] = (i < p && j < p) ? Rg[i + (int64_t)j * ldr] : 0.0; }
  __syncthreads();
  for (int j = threadIdx.x; j < p; j += blockDim.x) sInv[j] = 1.0 / sR[j + j * LD];
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r0 >= n) return;
  double x[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) x[j] = (j < p) ? (double)B[r0 + (int64_t)j * ldb] : 0.0;
#pragma unroll
  for (int j = 0; j < PB; ++j) {
    if (j < p) {
      double s = x[j];
      const double2* col = reinterpret_cast<const double2*>(sR + j * LD);
#pragma unroll
      for (int l2 = 0; l2 < (j + 1) / 2; ++l2) {
        const double2 rr = col[l2];
        s = fma(-x[2 * l2], rr.x, s);
        if (2 * l2 + 1 < j) s = fma(-x[2 * l2 + 1], rr.y, s);
      }
      x[j] = s * sInv[j];
    }
  }
#pragma unroll
  for (int j = 0; j < PB; ++j) if (j < p) Xo[r0 + (int64_t)j * ldx] = (float)x[j];
}
// V1: axpy form, LDS.128 row pairs, NaN-dependency against hoisting
template <int PB, int MINB>
__global__ void __launch_bounds__(256, MINB) v1(int64_t n, int p, const float* B, int64_t ldb, const double* __restrict__ Rg, int64_t ldr, float* Xo, int64_t ldx) {
  constexpr int LD = (PB + 1) & ~1;
  __shared__ __align__(16) double sR[PB * LD];
  __shared__ double sInv[PB];
  for (int e = threadIdx.x; e < LD * PB; e += blockDim.x) { const int j = e % LD, l = e / LD; sR[e] = (l < p && j < p && j >= l) ? Rg[l + (int64_t)j * ldr] : 0.0; }
  __syncthreads();
  for (int j = threadIdx.x; j < PB; j += blockDim.x) sInv[j] = j < p ? 1.0 / sR[j * LD + j] : 0.0;
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
  const float* pb = B + r;
#pragma unroll
  for (int j = 0; j < PB; ++j) { x[j] = j < p ? (double)*pb : 0.0; pb += ldb; }
  float* po = Xo + r;
#pragma unroll
  for (int l = 0; l < PB; ++l) {
    const double xl = x[l] * sInv[l];
    if (l < p) *po = (float)xl;
    po += ldx;
    const double2* row = reinterpret_cast<const double2*>(sR + l * LD + (xl != xl ? 2 : 0));
#pragma unroll
    for (int j2 = (l + 1) / 2; j2 < LD / 2; ++j2) {
      const double2 rr = row[j2];
      if (2 * j2 > l && 2 * j2 < PB) x[2 * j2] = fma(-xl, rr.x, x[2 * j2]);
      if (2 * j2 + 1 > l && 2 * j2 + 1 < PB) x[2 * j2 + 1] = fma(-xl, rr.y, x[2 * j2 + 1]);
    }
  }
}

// V2: dot form, G columns' chains interleaved (same per-column order, ILP G)
template <int PB, int G, int MINB>
__global__ void __launch_bounds__(256, MINB) v2(int64_t n, int p, const float* B, int64_t ldb, const double* __restrict__ Rg, int64_t ldr, float* Xo, int64_t ldx) {
  constexpr int LD = ((PB + G - 1) / G) * G;  // row-major R, rows padded to a multiple of G
  __shared__ __align__(16) double sR[PB * LD];
  __shared__ double sInv[PB];
  for (int e = threadIdx.x; e < LD * PB; e += blockDim.x) { const int j = e % LD, l = e / LD; sR[e] = (l < p && j < p && j >= l) ? Rg[l + (int64_t)j * ldr] : 0.0; }
  __syncthreads();
  for (int j = threadIdx.x; j < PB; j += blockDim.x) sInv[j] = j < p ? 1.0 / sR[j * LD + j] : 0.0;
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) x[j] = j < p ? (double)B[r + (int64_t)j * ldb] : 0.0;
#pragma unroll
  for (int j0 = 0; j0 < PB; j0 += G) {
    // chains of columns j0 .. j0+G-1 over the finished x_l, l < j0
#pragma unroll
    for (int l = 0; l < j0; ++l) {
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (j0 + g < PB) x[j0 + g] = fma(-x[l], sR[l * LD + j0 + g], x[j0 + g]);
    }
    // finish the panel in order
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (j0 + g < PB) {
#pragma unroll
        for (int h = 0; h < g; ++h) x[j0 + g] = fma(-x[j0 + h], sR[(j0 + h) * LD + j0 + g], x[j0 + g]);
        x[j0 + g] = x[j0 + g] * sInv[j0 + g];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < PB; ++j) if (j < p) Xo[r + (int64_t)j * ldx] = (float)x[j];
}

// V3: each row split over L = 4 lanes (columns j = t + 4 i), axpy order,
// x_l broadcast in the lane group by shuffle; same FMA order per column.
template <int PB, int MINB>
__global__ void __launch_bounds__(256, MINB) v3(int64_t n, int p, const float* B, int64_t ldb, const double* __restrict__ Rg, int64_t ldr, float* Xo, int64_t ldx) {
  constexpr int L = 4, NI = PB / L, TS = NI + 2;  // per-lane columns, padded lane stride
  __shared__ __align__(16) double sR[PB * L * TS];  // sR[(l * L + t) * TS + i] = R[l][t + 4 i] (j > l)
  __shared__ double sInv[PB];
  for (int e = threadIdx.x; e < PB * L * TS; e += blockDim.x) {
    const int i = e % TS, t = (e / TS) % L, l = e / (TS * L);
    const int j = t + L * i;
    sR[e] = (i < NI && l < p && j < p && j > l) ? Rg[l + (int64_t)j * ldr] : 0.0;
  }
  for (int j = threadIdx.x; j < PB; j += blockDim.x) sInv[j] = j < p ? 1.0 / Rg[j + (int64_t)j * ldr] : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, t = lane & (L - 1);
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
  const bool live = r < n;
  double x[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    const int j = t + L * i;
    x[i] = (live && j < p) ? (double)B[r + (int64_t)j * ldb] : 0.0;
  }
  const double* Rt = sR + t * TS;
#pragma unroll
  for (int l = 0; l < PB; ++l) {
    constexpr int dummy = 0; (void)dummy;
    const int io = l / L, o = l % L;
    double xl = 0.0;
    if (t == o) {
      xl = x[io] * sInv[l];
      x[io] = xl;
    }
    xl = __shfl_sync(0xffffffffu, xl, (lane & ~(L - 1)) | o);
    const double* Rl = Rt + l * L * TS;
    if (t > o) x[io] = fma(-xl, Rl[io], x[io]);
#pragma unroll
    for (int i = io + 1; i < NI; ++i) x[i] = fma(-xl, Rl[i], x[i]);
  }
  if (live) {
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int j = t + L * i;
      if (j < p) Xo[r + (int64_t)j * ldx] = (float)x[i];
    }
  }
}

// V4: R and 1/diag(R) in CONSTANT memory (loaded D2D per call), so every
// DFMA takes its R operand from the constant bank: no shared loads, no
// register writeback for R.  Dot form, same order as v0.
__constant__ double c_R[64 * 64];  // column-major, ld 64
__constant__ double c_inv[64];
template <int PB>
__global__ void __launch_bounds__(256, 2) v4(int64_t n, int p, const float* B, int64_t ldb, float* Xo, int64_t ldx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) x[j] = j < p ? (double)B[r + (int64_t)j * ldb] : 0.0;
#pragma unroll
  for (int j = 0; j < PB; ++j) {
    double s = x[j];
#pragma unroll
    for (int l = 0; l < j; ++l) s = fma(-x[l], c_R[l + j * 64], s);
    x[j] = s * c_inv[j];
  }
#pragma unroll
  for (int j = 0; j < PB; ++j) if (j < p) Xo[r + (int64_t)j * ldx] = (float)x[j];
}
__global__ void pack_R(int p, const double* R, int64_t ldr, double* Rp, double* inv) {
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int i = e % 64, j = e / 64;
    Rp[e] = (i < p && j < p) ? R[i + (int64_t)j * ldr] : 0.0;
  }
  for (int j = threadIdx.x; j < 64; j += blockDim.x) inv[j] = j < p ? 1.0 / R[j + (int64_t)j * ldr] : 0.0;
}

// V5: constant-bank R, axpy (right-looking) order: same FMA sequence per
// column as v0/v4, p-wide ILP.
template <int PB, int MINB>
__global__ void __launch_bounds__(256, MINB) v5(int64_t n, int p, const float* B, int64_t ldb, float* Xo, int64_t ldx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double x[PB];
#pragma unroll
  for (int j = 0; j < PB; ++j) x[j] = j < p ? (double)B[r + (int64_t)j * ldb] : 0.0;
#pragma unroll
  for (int l = 0; l < PB; ++l) {
    x[l] = x[l] * c_inv[l];
#pragma unroll
    for (int j = l + 1; j < PB; ++j) x[j] = fma(-x[l], c_R[l + j * 64], x[j]);
  }
#pragma unroll
  for (int j = 0; j < PB; ++j) if (j < p) Xo[r + (int64_t)j * ldx] = (float)x[j];
}
template <int PB>
void run(int64_t n) {
  const int p = PB;
  float *B, *X0, *X1; double* R;
  cudaMalloc(&B, n * p * 4); cudaMalloc(&X0, n * p * 4); cudaMalloc(&X1, n * p * 4); cudaMalloc(&R, p * p * 8);
  std::vector<double> h(p * p, 0.0);
  srand(3);
  for (int j = 0; j < p; ++j) for (int i = 0; i <= j; ++i) h[i + j * p] = (i == j) ? 1.0 + rand() / (double)RAND_MAX : 0.1 * (rand() / (double)RAND_MAX - 0.5);
  cudaMemcpy(R, h.data(), p * p * 8, cudaMemcpyHostToDevice);
  std::vector<float> hb(n * p); for (auto& v : hb) v = rand() / (float)RAND_MAX - 0.5f;
  cudaMemcpy(B, hb.data(), n * p * 4, cudaMemcpyHostToDevice);
  int grid = (int)((n + 255) / 256);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms[11];
  double* Rpk; cudaMalloc(&Rpk, (64 * 64 + 64) * 8);
  for (int v = 0; v < 11; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) {
        if (v == 0) v0<PB><<<grid, 256>>>(n, p, B, n, R, p, X0, n);
        else if (v == 1) v1<PB, 1><<<grid, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 2) v1<PB, 2><<<grid, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 3) v2<PB, 4, 2><<<grid, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 4) v2<PB, 8, 2><<<grid, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 5) v2<PB, 4, 1><<<grid, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 6) v3<PB, 2><<<grid * 4, 256>>>(n, p, B, n, R, p, X1, n);
        else if (v == 7) v3<PB, 4><<<grid * 4, 256>>>(n, p, B, n, R, p, X1, n);
        else {
          if (rep == 0 && v >= 8) {}
          pack_R<<<1, 256>>>(p, R, p, Rpk, Rpk + 64 * 64);
          cudaMemcpyToSymbolAsync(c_R, Rpk, 64 * 64 * 8, 0, cudaMemcpyDeviceToDevice);
          cudaMemcpyToSymbolAsync(c_inv, Rpk + 64 * 64, 64 * 8, 0, cudaMemcpyDeviceToDevice);
          if (v == 8) v4<PB><<<grid, 256>>>(n, p, B, n, X1, n);
          else if (v == 9) v5<PB, 2><<<grid, 256>>>(n, p, B, n, X1, n);
          else v5<PB, 1><<<grid, 256>>>(n, p, B, n, X1, n);
        }
      }
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[v], a, b); ms[v] /= 5;
    }
  }
  std::vector<float> o0(n * p), o1(n * p);
  cudaMemcpy(o0.data(), X0, n * p * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(o1.data(), X1, n * p * 4, cudaMemcpyDeviceToHost);
  int64_t diff = 0; for (int64_t i = 0; i < n * p; ++i) diff += memcmp(&o0[i], &o1[i], 4) != 0;
  printf("{\"p\": %d, \"n\": %lld, \"v0_ms\": %.4f, \"v1_minb1_ms\": %.4f, \"v1_minb2_ms\": %.4f, \"v2_g4_ms\": %.4f, \"v2_g8_ms\": %.4f, \"v2_g4_minb1_ms\": %.4f, \"v3_minb2_ms\": %.4f, \"v3_minb4_ms\": %.4f, \"v4_const_ms\": %.4f, \"v5_minb2_ms\": %.4f, \"v5_minb1_ms\": %.4f, \"bitdiff_last\": %lld, \"hbm_ms\": %.4f}\n", p, (long long)n, ms[0], ms[1], ms[2], ms[3], ms[4], ms[5], ms[6], ms[7], ms[8], ms[9], ms[10], (long long)diff, 2.0 * n * p * 4 / 6.5e12 * 1e3);
  cudaFree(B); cudaFree(X0); cudaFree(X1); cudaFree(R);
}
int main() {
  run<40>(1000000);
  run<64>(1 << 24);
  run<32>(1 << 24);
  return 0;
}
