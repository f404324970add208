// Instruction-throughput microbenchmarks for the design decisions in DESIGN.md
// (FMUL+FADD vs FFMA vs FFMA2 vs DFMA on sm_100a).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void kern(float* out, double* outd, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  double d0 = x0, d1 = x1, d2 = x2, d3 = x3, d4 = x4, d5 = x5, d6 = x6, d7 = x7;
  float2 p0 = make_float2(x0, x1), p1 = make_float2(x2, x3), p2 = make_float2(x4, x5), p3 = make_float2(x6, x7);
  float2 p4 = p0, p5 = p1, p6 = p2, p7 = p3;
  const float2 aa = make_float2(a, a), bb = make_float2(b, b);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) {  // FMUL + FADD (reference order), 8 independent chains
        x0 = __fadd_rn(x0, __fmul_rn(a, b + x1)); x1 = __fadd_rn(x1, __fmul_rn(a, x2)); x2 = __fadd_rn(x2, __fmul_rn(a, x3)); x3 = __fadd_rn(x3, __fmul_rn(a, x4));
        x4 = __fadd_rn(x4, __fmul_rn(a, x5)); x5 = __fadd_rn(x5, __fmul_rn(a, x6)); x6 = __fadd_rn(x6, __fmul_rn(a, x7)); x7 = __fadd_rn(x7, __fmul_rn(a, x0));
      } else if (OP == 1) {  // FFMA
        x0 = fmaf(a, x1, x0); x1 = fmaf(a, x2, x1); x2 = fmaf(a, x3, x2); x3 = fmaf(a, x4, x3);
        x4 = fmaf(a, x5, x4); x5 = fmaf(a, x6, x5); x6 = fmaf(a, x7, x6); x7 = fmaf(a, x0, x7);
      } else if (OP == 2) {  // FFMA2 (2 lanes each)
        p0 = __ffma2_rn(aa, p1, p0); p1 = __ffma2_rn(aa, p2, p1); p2 = __ffma2_rn(aa, p3, p2); p3 = __ffma2_rn(aa, p4, p3);
        p4 = __ffma2_rn(aa, p5, p4); p5 = __ffma2_rn(aa, p6, p5); p6 = __ffma2_rn(aa, p7, p6); p7 = __ffma2_rn(aa, p0, p7);
      } else if (OP == 3) {  // DFMA
        d0 = fma((double)a, d1, d0); d1 = fma((double)a, d2, d1); d2 = fma((double)a, d3, d2); d3 = fma((double)a, d4, d3);
        d4 = fma((double)a, d5, d4); d5 = fma((double)a, d6, d5); d6 = fma((double)a, d7, d6); d7 = fma((double)a, d0, d7);
      } else if (OP == 4) {  // DADD
        d0 = d0 + d1; d1 = d1 + d2; d2 = d2 + d3; d3 = d3 + d4; d4 = d4 + d5; d5 = d5 + d6; d6 = d6 + d7; d7 = d7 + d0;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + p0.x + p1.y + p2.x + p3.y + p4.x + p5.y + p6.x + p7.y;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = d0 + d1 + d2 + d3 + d4 + d5 + d6 + d7;
}

// fused vs separate check: does mul.rn.f32x2 + add.rn.f32x2 give separately rounded results?
__global__ void fusecheck(const float* q, const float* x, const float* w, float* o_sep, float* o_f2, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  o_sep[i] = __fadd_rn(w[i], __fmul_rn(q[i], x[i]));
  float2 r = __fadd2_rn(make_float2(w[i], w[i]), __fmul2_rn(make_float2(q[i], q[i]), make_float2(x[i], x[i])));
  o_f2[i] = r.x;
}

template <int OP>
double run(int blocks, int threads, int iters, float* o, double* od) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<OP><<<blocks, threads>>>(o, od, 10, 1.0000001f, 0.5f);
  cudaEventRecord(e0);
  kern<OP><<<blocks, threads>>>(o, od, iters, 1.0000001f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * 64;  // 8 unroll * 8 chains
  return ops / (ms * 1e-3);  // element-ops / s
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; double* od; cudaMalloc(&o, 1 << 26); cudaMalloc(&od, 1 << 27);
  int blocks = sms * 8, threads = 256, iters = 4096;
  const char* names[] = {"FMUL+FADD pair (elem/s)", "FFMA (elem/s)", "FFMA2 (instr/s, 2 elem each)", "DFMA (elem/s)", "DADD (elem/s)"};
  double r[5];
  r[0] = run<0>(blocks, threads, iters, o, od);
  r[1] = run<1>(blocks, threads, iters, o, od);
  r[2] = run<2>(blocks, threads, iters, o, od);
  r[3] = run<3>(blocks, threads, iters, o, od);
  r[4] = run<4>(blocks, threads, iters, o, od);
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  for (int i = 0; i < 5; ++i) printf(", \"%s\": %.4e, \"%s per SM per clk\": %.2f", names[i], r[i], names[i], r[i] / sms / (clk * 1e3));
  // fusion check
  const int n = 1 << 20;
  float *q, *x, *w, *a, *b;
  cudaMallocManaged(&q, n * 4); cudaMallocManaged(&x, n * 4); cudaMallocManaged(&w, n * 4); cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4);
  unsigned s = 1;
  for (int i = 0; i < n; ++i) { s = s * 1664525u + 1013904223u; q[i] = (s >> 8) * (1.0f / 16777216.0f) + 0.5f; s = s * 1664525u + 1013904223u; x[i] = -((s >> 8) * (1.0f / 16777216.0f) + 0.5f); s = s * 1664525u + 1013904223u; w[i] = (s >> 8) * (1.0f / 16777216.0f); }
  fusecheck<<<n / 256, 256>>>(q, x, w, a, b, n);
  cudaDeviceSynchronize();
  int diff = 0;
  for (int i = 0; i < n; ++i) diff += (a[i] != b[i]);
  printf(", \"f32x2 mul+add differs from separate (of 2^20)\": %d}\n", diff);
  return 0;
}
