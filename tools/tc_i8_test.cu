// Standalone check of the tcgen05 kind::i8 building blocks in csrc/tc.cuh:
// one CTA computes D (128 x 48, int32) = A (128 x 64, s8/u8) * B^T (48 x 64,
// s8/u8) with two K=32 MMAs and compares with a CPU product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_i8_test tools/tc_i8_test.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../paper_2111_14641_b200/csrc/tc.cuh"

using namespace rb::tc;

constexpr int M = 128, N = 48, K = 64;

template <bool AS, bool BS>
__global__ void kern(const uint8_t* A, const uint8_t* B, int* D) {
  __shared__ __align__(128) uint8_t sA[M * K];  // [kc][row][16]
  __shared__ __align__(128) uint8_t sB[N * K];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x;
  for (int e = t; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    sA[(k / 16) * (M * 16) + r * 16 + (k % 16)] = A[r * K + k];
  }
  for (int e = t; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    sB[(k / 16) * (N * 16) + r * 16 + (k % 16)] = B[r * K + k];
  }
  if (t == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (t < 32) tmem_alloc(&tbase, 64);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t d = tbase;
  if (t == 0) {
    const uint32_t id = idesc_i8(M, N, AS, BS);
    for (int ks = 0; ks < K / 32; ++ks) {
      const uint64_t a = sdesc_kmajor(smem_u32(sA) + ks * 2 * (M * 16), M * 16, 128);
      const uint64_t b = sdesc_kmajor(smem_u32(sB) + ks * 2 * (N * 16), N * 16, 128);
      mma_i8(d, a, b, id, ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int w = t >> 5;
  uint32_t r[16];
  for (int c0 = 0; c0 < N; c0 += 16) {
    tmem_ld16(d + ((uint32_t)(32 * w) << 16) + c0, r);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(32 * w + (t & 31)) * N + c0 + j] = (int)r[j];
  }
  tc_fence_before();
  __syncthreads();
  if (t < 32) tmem_dealloc(tbase, 64);
}

template <bool AS, bool BS>
int run() {
  uint8_t *A, *B;
  int* D;
  cudaMallocManaged(&A, M * K);
  cudaMallocManaged(&B, N * K);
  cudaMallocManaged(&D, M * N * 4);
  srand(AS * 2 + BS + 1);
  for (int i = 0; i < M * K; ++i) A[i] = rand() & 255;
  for (int i = 0; i < N * K; ++i) B[i] = rand() & 255;
  kern<AS, BS><<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("cuda error %s\n", cudaGetErrorString(e));
    return 1;
  }
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < K; ++k) {
        const int a = AS ? (int)(int8_t)A[i * K + k] : (int)A[i * K + k];
        const int b = BS ? (int)(int8_t)B[j * K + k] : (int)B[j * K + k];
        s += a * b;
      }
      if (s != D[i * N + j]) {
        if (bad < 5) printf("  mismatch (%d,%d): gpu %d cpu %ld\n", i, j, D[i * N + j], s);
        ++bad;
      }
    }
  printf("a_signed=%d b_signed=%d: %d mismatches of %d\n", AS, BS, bad, M * N);
  return bad != 0;
}

int main() {
  int f = 0;
  f |= run<true, true>();
  f |= run<true, false>();
  f |= run<false, true>();
  f |= run<false, false>();
  printf(f ? "FAIL\n" : "PASS\n");
  return f;
}
