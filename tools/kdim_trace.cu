// Phase timeline of the cooperative k-dimensional kernels: kdim.cu built
// with RB_KDIM_TRACE (CTA 0 stamps %globaltimer at phase boundaries).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/kdim_trace.cu -o tools/kdim_trace
#define RB_KDIM_TRACE 1
#include <cstdarg>
#include <cstdio>
#include <vector>

#include "../paper_2111_14641_b200/csrc/kdim.cu"

namespace rb {
unsigned long long g_launches = 0;
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfprintf(stderr, fmt, ap);
  va_end(ap);
  fprintf(stderr, "\n");
}
int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); return RB_ECUDA; }
  return RB_OK;
}
int sm_count() {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0);
  return v;
}
}  // namespace rb

__global__ void chase(const double* ring, int n, double* out) {
  unsigned long long t0, t1;
  double v = 0.0;
  int idx = 0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < n; ++i) {
    v = __ldcg(&ring[idx]);
    idx = (int)v;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  g_kdim_trace[200] = t0;
  g_kdim_trace[201] = t1;
  out[0] = v;
}

static void dump(const char* name, std::vector<int> slots) {
  unsigned long long t[256];
  cudaMemcpyFromSymbol(t, g_kdim_trace, sizeof(t));
  printf("%s:", name);
  unsigned long long t0 = t[slots[0]];
  for (int s : slots) printf(" %d:%.2f", s, (t[s] - t0) * 1e-3);
  printf("  (us)\n");
}

int main() {
  const int k = 1600, c = 760, p = 40, l = 5;
  std::vector<double> h((size_t)k * c);
  for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
  double *S, *P, *X, *T, *R, *So, *ws;
  int* info;
  cudaMalloc(&S, h.size() * 8);
  cudaMalloc(&P, (size_t)k * p * 8);
  cudaMalloc(&X, (size_t)c * p * 8);
  cudaMalloc(&T, (size_t)k * p * 8);
  cudaMalloc(&R, p * p * 8);
  cudaMalloc(&So, (size_t)k * p * 8);
  cudaMalloc(&info, 4);
  size_t wsb = 64 << 20;
  cudaMalloc(&ws, wsb);
  cudaMemcpy(S, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(P, h.data(), (size_t)k * p * 8, cudaMemcpyHostToDevice);
  for (int cc : {760, 380, 40}) {
    for (int rep = 0; rep < 3; ++rep) rb::ls_richardson(k, cc, p, S, k, P, k, l, X, c, T, k, ws, wsb, 0);
    cudaDeviceSynchronize();
    char nm[64];
    snprintf(nm, sizeof nm, "richardson c=%d", cc);
    std::vector<int> sl;
    for (int i = 0; i <= 8 * (l - 1) + 8; ++i) sl.push_back(i);
    dump(nm, sl);
  }
  for (int rep = 0; rep < 3; ++rep) rb::sketched_cholqr_small(k, p, P, k, R, p, So, k, info, ws, wsb, 0);
  cudaDeviceSynchronize();
  dump("cholqr", {100, 110, 101, 102, 103, 104, 105, 106});
  // raw L2 round trip: one thread, dependent loads over a 1 MB ring already in L2
  {
    double* ring;
    cudaMalloc(&ring, 1 << 20);
    std::vector<double> hr(1 << 17);
    for (size_t i = 0; i < hr.size(); ++i) hr[i] = (double)((i * 7919 + 4096) % hr.size());
    cudaMemcpy(ring, hr.data(), 1 << 20, cudaMemcpyHostToDevice);
    chase<<<1, 1>>>(ring, 1000, ws);
    chase<<<1, 1>>>(ring, 1000, ws);
    cudaDeviceSynchronize();
    unsigned long long tt[256];
    cudaMemcpyFromSymbol(tt, g_kdim_trace, sizeof(tt));
    printf("L2 dependent-load latency: %.1f ns\n", (tt[201] - tt[200]) / 1000.0);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
