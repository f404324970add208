#include <cstdio>
__global__ void k(const double* a, const double* b, double* c, int iters) {
  double a0 = a[threadIdx.x], a1 = a[threadIdx.x + 32], b0 = b[threadIdx.x];
  double d[4] = {0, 0, 0, 0};
  double e[4] = {0, 0, 0, 0};
  for (int i = 0; i < iters; ++i) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(e[0]), "+d"(e[1]), "+d"(e[2]), "+d"(e[3]) : "d"(a1), "d"(a0), "d"(b0));
  }
  c[blockIdx.x * 128 + threadIdx.x] = d[0] + d[1] + d[2] + d[3] + e[0] + e[1] + e[2] + e[3];
}
__global__ void kf(const double* a, const double* b, double* c, int iters) {
  double x = a[threadIdx.x], y = b[threadIdx.x];
  double acc[16];
  for (int q = 0; q < 16; ++q) acc[q] = q;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = fma(x, y, acc[q]);
  double s = 0;
  for (int q = 0; q < 16; ++q) s += acc[q];
  c[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *a, *b, *c;
  cudaMalloc(&a, 1 << 20); cudaMalloc(&b, 1 << 20); cudaMalloc(&c, 64 << 20);
  cudaMemset(a, 0, 1 << 20); cudaMemset(b, 0, 1 << 20);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int w : {4, 8, 16}) {
    k<<<148, 32 * w>>>(a, b, c, iters);
    cudaEventRecord(e0);
    k<<<148, 32 * w>>>(a, b, c, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * w * iters * 2 * 512;
    printf("DMMA m16n8k4 warps/SM %d: %.2f TFLOP/s (fp64)\n", w, 2 * fma / (ms * 1e-3) / 1e12);
  }
  for (int t : {256, 512, 1024}) {
    kf<<<148, t>>>(a, b, c, iters);
    cudaEventRecord(e0);
    kf<<<148, t>>>(a, b, c, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * t * iters * 16;
    printf("DFMA threads/SM %d: %.2f TFLOP/s (fp64)\n", t, 2 * fma / (ms * 1e-3) / 1e12);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
