#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
// does ffma2(q,x,z) [z = runtime -0] + fadd2(acc, prod) stay separately rounded?
__global__ void fusecheck(const float* q, const float* x, const float* w, float* o_sep, float* o_pk, int n, float z) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  o_sep[i] = __fadd_rn(w[i], __fmul_rn(q[i], x[i]));
  float2 zz = make_float2(z, z);
  float2 pr = __ffma2_rn(make_float2(q[i], q[i]), make_float2(x[i], -x[i]), zz);
  float2 r = __fadd2_rn(make_float2(w[i], w[i]), pr);
  o_pk[i] = r.x;
}
// throughput: chains like the projection step, packed vs scalar
template <bool PK>
__global__ void thr(float* out, int iters, float z, float a0) {
  float acc[32];
  for (int j = 0; j < 32; ++j) acc[j] = threadIdx.x * 1e-3f + j;
  float q = a0 + threadIdx.x * 1e-7f;
  const float2 zz = make_float2(z, z);
  for (int it = 0; it < iters; ++it) {
    q = q * 0.999f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) {
      if (PK) {
        float2 pr = __ffma2_rn(make_float2(q, q), make_float2(acc[j+1], acc[j]), zz);
        float2 s = __fadd2_rn(make_float2(acc[j], acc[j+1]), pr);
        acc[j] = s.x; acc[j+1] = s.y;
      } else {
        acc[j] = __fadd_rn(acc[j], __fmul_rn(q, acc[j+1]));
        acc[j+1] = __fadd_rn(acc[j+1], __fmul_rn(q, acc[j]));
      }
    }
  }
  float s = 0; for (int j = 0; j < 32; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  const int n = 1 << 20;
  float *q, *x, *w, *a, *b;
  cudaMallocManaged(&q, n * 4); cudaMallocManaged(&x, n * 4); cudaMallocManaged(&w, n * 4);
  cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4);
  srand(1);
  for (int i = 0; i < n; ++i) { q[i] = (rand() / (float)RAND_MAX - 0.5f) * 3; x[i] = (rand() / (float)RAND_MAX - 0.5f) * 7; w[i] = (rand() / (float)RAND_MAX - 0.5f); if (i % 97 == 0) w[i] = -0.0f; if (i%89==0) q[i]=0.f;}
  fusecheck<<<n / 256, 256>>>(q, x, w, a, b, n, -0.0f);
  cudaDeviceSynchronize();
  int diff = 0; for (int i = 0; i < n; ++i) if (memcmp(&a[i], &b[i], 4)) ++diff;
  printf("{\"packed ffma2(-0)+fadd2 bit diffs of 2^20\": %d", diff);
  float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int pk = 0; pk < 2; ++pk) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (pk) thr<true><<<148 * 8, 256>>>(o, iters, -0.0f, 1.0f); else thr<false><<<148 * 8, 256>>>(o, iters, -0.0f, 1.0f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double elem = 148.0 * 8 * 256 * iters * 32;
      if (rep) printf(", \"%s elem-steps/s\": %.4g", pk ? "packed" : "scalar", elem / ms * 1e3);
    }
  }
  printf("}\n");
  return 0;
}
