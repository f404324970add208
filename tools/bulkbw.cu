// Microbenchmark: HBM -> shared memory streaming with cp.async.bulk (1-D TMA)
// on one CTA per SM, varying the copy size and the number of stages in
// flight.  Decides the pipeline shape of sketch_tc.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bulkbw tools/bulkbw.cu
#include <cstdio>
#include <cstdint>

#include "../paper_2111_14641_b200/csrc/tc.cuh"

using namespace rb::tc;

__global__ void stream(const uint8_t* src, size_t per_cta, int copy_bytes, int stages, int split, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[8];
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const int tiles = (int)(per_cta / copy_bytes);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned acc = 0;
    const int piece = copy_bytes / split;
    for (int t = 0; t < tiles + stages; ++t) {
      if (t >= stages) {
        const int s = (t - stages) % stages;
        mbar_wait(&full[s], ((t - stages) / stages) & 1);
        acc += sm[s * copy_bytes];
      }
      if (t < tiles) {
        const int s = t % stages;
        mbar_arrive_expect_tx(&full[s], copy_bytes);
        for (int q = 0; q < split; ++q)
          bulk_g2s(sm + s * copy_bytes + q * piece, base + (size_t)t * copy_bytes + q * piece, piece, &full[s]);
      }
    }
    sink[blockIdx.x] = acc;
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t per_cta = (size_t)24 << 20;  // 24 MB per CTA
  uint8_t* src;
  unsigned* sink;
  cudaMalloc(&src, per_cta * sms);
  cudaMemset(src, 1, per_cta * sms);
  cudaMalloc(&sink, sms * 4);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int sizes[] = {8192, 16384, 32768, 65536};
  const int stg[] = {2, 3, 4, 6, 8};
  const int splits[] = {1, 4};
  printf("{");
  bool first = true;
  for (int sz : sizes)
    for (int st : stg)
      for (int sp : splits) {
        if ((size_t)sz * st > 216 * 1024) continue;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        stream<<<sms, 32, sz * st>>>(src, per_cta, sz, st, sp, sink);
        cudaEventRecord(a);
        stream<<<sms, 32, sz * st>>>(src, per_cta, sz, st, sp, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = per_cta * sms / (ms * 1e-3) / 1e9;
        printf("%s\"size%d_st%d_split%d\": %.1f", first ? "" : ", ", sz, st, sp, gbs);
        first = false;
      }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
